// micro-benchmark: decode variants throughput (fields from shared memory)
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ double decA(uint32_t lo, uint32_t hi, unsigned s, uint32_t mask, uint32_t mul, uint64_t bias) {
    const uint32_t t = __funnelshift_l(lo, hi, s);
    const uint64_t bits = static_cast<uint64_t>(t & mask) * mul + bias;
    const double v = __longlong_as_double(static_cast<long long>(bits)) - 1.0;
    return __hiloint2double(__double2hiint(v) ^ static_cast<int>(t & 0x80000000u), __double2loint(v));
}
__device__ __forceinline__ double decB(uint32_t lo, uint32_t hi, unsigned s, uint32_t mask, uint32_t mul, uint32_t biashi) {
    const uint32_t t = __funnelshift_l(lo, hi, s);
    const uint32_t h = __umulhi(t & mask, mul) + biashi;
    const double v = __hiloint2double(static_cast<int>(h), 0) - 1.0;
    return __hiloint2double(__double2hiint(v) ^ static_cast<int>(t & 0x80000000u), __double2loint(v));
}
__device__ __forceinline__ double decC(uint32_t lo, uint32_t hi, unsigned s, uint32_t mask, uint32_t mul, uint64_t bias) {
    const uint32_t t = __funnelshift_l(lo, hi, s);
    const uint64_t bits = static_cast<uint64_t>(t & mask) * mul + bias;
    return __longlong_as_double(static_cast<long long>(bits));  // no -1, no sign (timing only)
}
__device__ __forceinline__ double decD(uint32_t lo, uint32_t hi, unsigned s, uint32_t mask, uint32_t mul, uint64_t bias) {
    const uint32_t t = __funnelshift_l(lo, hi, s);
    const uint64_t bits = static_cast<uint64_t>(t & mask) * mul + bias;
    return __longlong_as_double(static_cast<long long>(bits)) - 1.0;  // no sign (timing only)
}
template <int V>
__global__ void k(const uint32_t* g, double* out, int iters, uint32_t mask, uint32_t mul, uint64_t bias) {
    __shared__ uint4 sm[1026];
    for (int i = threadIdx.x; i < 1026; i += blockDim.x) sm[i] = make_uint4(g[i], g[i+1], g[i+2], g[i+3]);
    __syncthreads();
    double acc[4] = {0, 0, 0, 0};
    double acc2[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const unsigned s = 0u - (threadIdx.x * 7u + 13u);
    int o = threadIdx.x & 511;
    for (int it = 0; it < iters; ++it) {
        const uint4 a = sm[o], b = sm[o + 1];
        const double x = 1.0 + it * 1e-9;
        if (V == 2) {
            acc[0] = fma(decC(a.x, b.x, s, mask, mul, bias), x, acc[0]);
            acc[1] = fma(decC(a.y, b.y, s, mask, mul, bias), x, acc[1]);
            acc[2] = fma(decC(a.z, b.z, s, mask, mul, bias), x, acc[2]);
            acc[3] = fma(decC(a.w, b.w, s, mask, mul, bias), x, acc[3]);
        } else if (V == 3) {
            acc[0] = fma(decD(a.x, b.x, s, mask, mul, bias), x, acc[0]);
            acc[1] = fma(decD(a.y, b.y, s, mask, mul, bias), x, acc[1]);
            acc[2] = fma(decD(a.z, b.z, s, mask, mul, bias), x, acc[2]);
            acc[3] = fma(decD(a.w, b.w, s, mask, mul, bias), x, acc[3]);
        } else if (V == 4) {  // 8 chains: alternate accumulator sets
            const int h = (it & 1) * 4;
            acc2[h + 0] = fma(decA(a.x, b.x, s, mask, mul, bias), x, acc2[h + 0]);
            acc2[h + 1] = fma(decA(a.y, b.y, s, mask, mul, bias), x, acc2[h + 1]);
            acc2[h + 2] = fma(decA(a.z, b.z, s, mask, mul, bias), x, acc2[h + 2]);
            acc2[h + 3] = fma(decA(a.w, b.w, s, mask, mul, bias), x, acc2[h + 3]);
        } else if (V == 5) {  // 8 independent fields per iteration (two quads)
            const uint4 c = sm[(o + 256) & 1023], d = sm[((o + 256) & 1023) + 1];
            acc2[0] = fma(decA(a.x, b.x, s, mask, mul, bias), x, acc2[0]);
            acc2[1] = fma(decA(a.y, b.y, s, mask, mul, bias), x, acc2[1]);
            acc2[2] = fma(decA(a.z, b.z, s, mask, mul, bias), x, acc2[2]);
            acc2[3] = fma(decA(a.w, b.w, s, mask, mul, bias), x, acc2[3]);
            acc2[4] = fma(decA(c.x, d.x, s, mask, mul, bias), x, acc2[4]);
            acc2[5] = fma(decA(c.y, d.y, s, mask, mul, bias), x, acc2[5]);
            acc2[6] = fma(decA(c.z, d.z, s, mask, mul, bias), x, acc2[6]);
            acc2[7] = fma(decA(c.w, d.w, s, mask, mul, bias), x, acc2[7]);
        } else if (V == 0) {
            acc[0] = fma(decA(a.x, b.x, s, mask, mul, bias), x, acc[0]);
            acc[1] = fma(decA(a.y, b.y, s, mask, mul, bias), x, acc[1]);
            acc[2] = fma(decA(a.z, b.z, s, mask, mul, bias), x, acc[2]);
            acc[3] = fma(decA(a.w, b.w, s, mask, mul, bias), x, acc[3]);
        } else {
            const uint32_t bh = static_cast<uint32_t>(bias >> 32);
            acc[0] = fma(decB(a.x, b.x, s, mask, mul, bh), x, acc[0]);
            acc[1] = fma(decB(a.y, b.y, s, mask, mul, bh), x, acc[1]);
            acc[2] = fma(decB(a.z, b.z, s, mask, mul, bh), x, acc[2]);
            acc[3] = fma(decB(a.w, b.w, s, mask, mul, bh), x, acc[3]);
        }
        o = (o + 5) & 511;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc[0] + acc[1] + acc[2] + acc[3] + acc2[0] + acc2[1] + acc2[2] + acc2[3] + acc2[4] + acc2[5] + acc2[6] + acc2[7];
}
int main() {
    uint32_t* g; double* out;
    cudaMalloc(&g, 8192 * 4); cudaMemset(g, 0x5a, 8192 * 4);
    cudaMalloc(&out, 148 * 8 * 1024 * 8);
    const unsigned w = 24, e = 4;
    const uint32_t mask = 0x7fffffffu & ~((0xffffffffu >> (w - 1)) >> 1), mul = 1u << (21 + e);
    const uint64_t bias = 1023ull << 52;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int wpb : {8, 16}) {
      for (int v = 0; v < 6; ++v) {
        int iters = 4096;
        auto run = [&]{ switch (v) { case 0: k<0><<<148 * 2, wpb * 32>>>(g, out, iters, mask, mul, bias); break;
            case 1: k<1><<<148 * 2, wpb * 32>>>(g, out, iters, mask, mul, bias); break;
            case 2: k<2><<<148 * 2, wpb * 32>>>(g, out, iters, mask, mul, bias); break;
            case 3: k<3><<<148 * 2, wpb * 32>>>(g, out, iters, mask, mul, bias); break;
            case 4: k<4><<<148 * 2, wpb * 32>>>(g, out, iters, mask, mul, bias); break;
            default: k<5><<<148 * 2, wpb * 32>>>(g, out, iters, mask, mul, bias); break; } };
        run(); cudaDeviceSynchronize();
        cudaEventRecord(e0); run(); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double fields = 148.0 * 2 * wpb * 32 * iters * (v == 5 ? 8 : 4);
        printf("warps/CTA %2d variant %d: %.3f ms, %.1f G fields/s\n", wpb, v, ms, fields / ms / 1e6);
      }
    }
    return 0;
}
