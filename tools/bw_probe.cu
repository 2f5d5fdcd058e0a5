// Bandwidth probe (not part of the product): how fast can a CTA-level
// cp.async.bulk ring stream HBM through shared memory on this B200, with and
// without extra small copies per stage, vs plain LDG.128 reads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bw_probe tools/bw_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* b, unsigned n) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, unsigned ph) {
    asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(sa(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, unsigned n, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(d)), "l"(s), "r"(n), "r"(sa(b)) : "memory");
}

template <int NW, int STAGE, int NS, int NSMALL>
__global__ void __launch_bounds__((NW + 1) * 32) k_ring(const uint8_t* src, size_t per_cta, const uint8_t* small, unsigned* sink) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint64_t* full = (uint64_t*)(sm + NS * (STAGE + NSMALL * 256));
    uint64_t* empty = full + NS;
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint8_t* base = src + blockIdx.x * per_cta;
    const unsigned nst = per_cta / STAGE;
    if (tid == 0) {
        for (int i = 0; i < NS; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], NW); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == NW) {
        for (unsigned s = 0; s < nst; ++s) {
            const int slot = s % NS;
            if (s >= NS) wait(&empty[slot], ((s / NS) - 1) & 1);
            uint8_t* dst = sm + slot * (STAGE + NSMALL * 256);
            if (lane == 0) {
                expect_tx(&full[slot], STAGE + NSMALL * 256);
                bulk(dst, base + (size_t)s * STAGE, STAGE, &full[slot]);
            }
            __syncwarp();
            if (lane < NSMALL) bulk(dst + STAGE + lane * 256, small + ((s * 7 + lane) % 1024) * 256, 256, &full[slot]);
        }
        return;
    }
    unsigned acc = 0;
    for (unsigned s = 0; s < nst; ++s) {
        const int slot = s % NS;
        wait(&full[slot], (s / NS) & 1);
        const uint32_t* w = (const uint32_t*)(sm + slot * (STAGE + NSMALL * 256));
        for (unsigned i = warp * 32 + lane; i < STAGE / 4; i += NW * 32) acc += w[i];
        __syncwarp();
        if (lane == 0) arrive(&empty[slot]);
    }
    if (acc == 0x12345678) sink[0] = acc;
}

__global__ void k_ldg(const uint4* src, size_t n, unsigned* sink) {
    unsigned acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint4 v = __ldcs(src + i);
        acc += v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678) sink[0] = acc;
}

template <int NW, int STAGE, int NS, int NSMALL>
void run(const uint8_t* d, size_t bytes, const uint8_t* small, unsigned* sink, int ctas_per_sm, const char* name) {
    auto k = k_ring<NW, STAGE, NS, NSMALL>;
    const size_t smem = NS * (STAGE + NSMALL * 256) + 2 * NS * 8;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = 148 * ctas_per_sm;
    const size_t per = (bytes / grid) / STAGE * STAGE;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int it = 0; it < 2; ++it) k<<<grid, (NW + 1) * 32, smem>>>(d, per, small, sink);
    cudaEventRecord(a);
    for (int it = 0; it < 5; ++it) k<<<grid, (NW + 1) * 32, smem>>>(d, per, small, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%-48s ctas/SM=%d smem=%zu KB: %.1f GB/s (%s)\n", name, ctas_per_sm, smem / 1024,
           5.0 * per * grid / (ms / 1e3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const size_t bytes = 2ull << 30;
    uint8_t *d, *small; unsigned* sink;
    cudaMalloc(&d, bytes); cudaMemset(d, 1, bytes);
    cudaMalloc(&small, 1 << 20); cudaMemset(small, 2, 1 << 20);
    cudaMalloc(&sink, 4);
    {
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        k_ldg<<<148 * 8, 512>>>((const uint4*)d, bytes / 16, sink);
        cudaEventRecord(a);
        for (int i = 0; i < 5; ++i) k_ldg<<<148 * 8, 512>>>((const uint4*)d, bytes / 16, sink);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("LDG.128 read: %.1f GB/s\n", 5.0 * bytes / (ms / 1e3) / 1e9);
    }
    run<16, 24576, 3, 0>(d, bytes, small, sink, 2, "ring 24KB x3, 16 warps");
    run<16, 24576, 4, 0>(d, bytes, small, sink, 2, "ring 24KB x4, 16 warps");
    run<16, 24576, 3, 16>(d, bytes, small, sink, 2, "ring 24KB x3 + 16 small copies");
    run<16, 24576, 3, 32>(d, bytes, small, sink, 2, "ring 24KB x3 + 32 small copies");
    run<8, 16384, 6, 0>(d, bytes, small, sink, 2, "ring 16KB x6, 8 warps");
    run<8, 32768, 3, 0>(d, bytes, small, sink, 2, "ring 32KB x3, 8 warps");
    run<8, 8192, 8, 0>(d, bytes, small, sink, 3, "ring 8KB x8, 8 warps");
    run<4, 4096, 8, 0>(d, bytes, small, sink, 6, "ring 4KB x8, 4 warps");
    run<16, 49152, 2, 0>(d, bytes, small, sink, 2, "ring 48KB x2");
    run<16, 65536, 3, 0>(d, bytes, small, sink, 1, "ring 64KB x3, 1 CTA");
    return 0;
}
