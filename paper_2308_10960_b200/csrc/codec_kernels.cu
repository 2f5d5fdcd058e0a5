// codec_kernels.cu -- sm_100a kernels of the adaptive-precision codec and the
// batched / host-pointer codec entry points of the C-ABI.
//
//   k_analyze  : codec.cpp:44-60  analyze (per-buffer min/max of nonzero |v|)
//   k_pack     : codec.cpp:103-140 compress_block + BitWriter (bitstream.hpp:19-59)
//   k_unpack   : codec.cpp:146-171 decompress_into + BitReader (bitstream.hpp:63-97)
//
// Work unit: one warp per "job" = up to 512 groups of 32 consecutive values of
// one buffer.  A group of 32 values at bit width w occupies exactly w 32-bit
// words of the LSB-first stream, so groups are independent: no atomics between
// warps when packing, and each group's words are written once, coalesced.
//
// Bit-exactness: the encoder computes |v| * (1/scale) + 1 as two correctly
// rounded operations (__dmul_rn, __dadd_rn: the reference's Release build has no
// FMA at codec.cpp:124), and 1/scale with IEEE division.  Decoding is
// exact by construction ((1.mant * 2^off) - 1 is exact, one rounding in * scale).
#include <atomic>
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <vector>

#include "internal.h"

namespace hcmx_gpu {

void check_cuda(int err, const char* what) {
    if (err != cudaSuccess) {
        cudaGetLastError();
        throw cuda_error(std::string(what) + ": " + cudaGetErrorString(static_cast<cudaError_t>(err)));
    }
}

void require_device() {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        throw cuda_error("no CUDA device: libhcmx_gpu has no CPU fallback");
    }
}

// Small device buffers (job lists, descriptors, offsets) come from a
// process-wide cache of power-of-two blocks: cudaMalloc/cudaFree synchronise
// the device and cost more than the kernels of a batched codec call.  Every
// user of a cached block synchronises its stream before releasing it.
namespace {
constexpr size_t kPoolMax = size_t(64) << 20;
std::mutex g_pool_mu;
std::vector<std::vector<void*>> g_pool(40);
int size_class(size_t n) {
    int c = 8;  // 256 B minimum
    while ((size_t(1) << c) < n) ++c;
    return c;
}
}  // namespace

void DevBuf::alloc(size_t n) {
    release();
    if (n == 0) return;
    if (n <= kPoolMax) {
        const int c = size_class(n);
        {
            std::lock_guard<std::mutex> g(g_pool_mu);
            if (!g_pool[c].empty()) {
                p = g_pool[c].back();
                g_pool[c].pop_back();
                bytes = n;
                return;
            }
        }
        n = size_t(1) << c;
    }
    cudaError_t e = cudaMalloc(&p, n);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        p = nullptr;
        throw oom_error("cudaMalloc failed (out of device memory)");
    }
    check_cuda(e, "cudaMalloc");
    bytes = n;
}

void DevBuf::release() {
    if (p) {
        if (bytes <= kPoolMax) {
            std::lock_guard<std::mutex> g(g_pool_mu);
            g_pool[size_class(bytes)].push_back(p);
        } else {
            cudaFree(p);
        }
    }
    p = nullptr;
    bytes = 0;
}

void h2d(void* dst, const void* src, size_t bytes, void* stream) {
    if (!bytes) return;
    check_cuda(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, (cudaStream_t)stream), "h2d");
}
void d2h(void* dst, const void* src, size_t bytes, void* stream) {
    if (!bytes) return;
    check_cuda(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, (cudaStream_t)stream), "d2h");
}
void stream_sync(void* stream) {
    check_cuda(cudaStreamSynchronize((cudaStream_t)stream), "cudaStreamSynchronize");
}

namespace {

constexpr unsigned kGroupsPerJob = 32;  // 1024 values per warp job
constexpr uint64_t kFuseMax = 1ull << 17;  // fused compress: one warp per buffer up to this size
constexpr int kWarpsPerBlock = 8;
// occupancy knobs (resident CTAs per SM asked of ptxas) of the unpack and register-resident compress kernels
#ifndef HCMX_UNPACK_MINB
#define HCMX_UNPACK_MINB 1
#endif
#ifndef HCMX_COMPRESS_KIND
#define HCMX_COMPRESS_KIND 0  // buffers <= 4096 values: 0 TMA-staged, 1 register-resident, 2 two-pass CTA
#endif
#ifndef HCMX_REG_MINB
#define HCMX_REG_MINB 1
#endif

struct Job {
    uint32_t buf;
    uint32_t g0;
    uint32_t ng;
    uint32_t pad;
};

std::vector<Job> make_jobs(const uint64_t* count, uint64_t nbuf) {
    std::vector<Job> jobs;
    jobs.reserve(nbuf);
    for (uint64_t b = 0; b < nbuf; ++b) {
        const uint64_t groups = (count[b] + 31) / 32;
        for (uint64_t g = 0; g < groups; g += kGroupsPerJob)
            jobs.push_back({static_cast<uint32_t>(b), static_cast<uint32_t>(g),
                            static_cast<uint32_t>(std::min<uint64_t>(kGroupsPerJob, groups - g)), 0});
    }
    return jobs;
}

__device__ __forceinline__ uint64_t dbits(double d) { return static_cast<uint64_t>(__double_as_longlong(d)); }
__device__ __forceinline__ double bitsd(uint64_t u) { return __longlong_as_double(static_cast<long long>(u)); }
__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

// ------------------------------------------------------------ analyze ----
__global__ void k_stats_init(hcmx_stats* st, uint64_t nbuf) {
    for (uint64_t b = blockIdx.x * blockDim.x + threadIdx.x; b < nbuf; b += gridDim.x * blockDim.x) {
        reinterpret_cast<unsigned long long*>(&st[b].min_mag)[0] = 0x7FF0000000000000ull;  // +inf
        reinterpret_cast<unsigned long long*>(&st[b].max_mag)[0] = 0ull;
        st[b].all_zero = 1u;
        st[b].non_finite = 0u;
    }
}

// codec.cpp:44-60: min/max over nonzero |v|.  NaN counts as nonzero but never
// wins std::min/std::max there; the same holds below (NaN compares false).
__global__ void k_analyze(const double* __restrict__ values, const uint64_t* __restrict__ voff,
                          const uint64_t* __restrict__ count, const Job* __restrict__ jobs,
                          uint64_t njobs, hcmx_stats* st) {
    const unsigned lane = threadIdx.x & 31;
    const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    for (uint64_t j = wid; j < njobs; j += nw) {
        const Job jb = jobs[j];
        const uint64_t n = count[jb.buf];
        const uint64_t i0 = (uint64_t)jb.g0 * 32, i1 = umin64(n, (uint64_t)(jb.g0 + jb.ng) * 32);
        const double* v = values + voff[jb.buf];
        uint64_t mn = 0x7FF0000000000000ull, mx = 0;
        unsigned nz = 0, nf = 0;
        for (uint64_t i = i0 + lane; i < i1; i += 128) {
            double xs[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) xs[u] = i + 32 * u < i1 ? __ldcs(v + i + 32 * u) : 0.0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const double x = xs[u];
                const double a = fabs(x);
                if (a != 0.0) nz = 1;
                if (!isfinite(x)) nf = 1;
                if (a != 0.0 && !isnan(a)) {
                    const uint64_t b = dbits(a);  // nonnegative doubles order like their bits
                    mn = b < mn ? b : mn;
                    mx = b > mx ? b : mx;
                }
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const uint64_t omn = __shfl_xor_sync(0xffffffffu, mn, o);
            const uint64_t omx = __shfl_xor_sync(0xffffffffu, mx, o);
            mn = omn < mn ? omn : mn;
            mx = omx > mx ? omx : mx;
        }
        nz = __any_sync(0xffffffffu, nz);
        nf = __any_sync(0xffffffffu, nf);
        if (lane == 0) {
            hcmx_stats* s = st + jb.buf;
            atomicMin(reinterpret_cast<unsigned long long*>(&s->min_mag), (unsigned long long)mn);
            atomicMax(reinterpret_cast<unsigned long long*>(&s->max_mag), (unsigned long long)mx);
            if (nz) atomicAnd(&s->all_zero, 0u);
            if (nf) atomicOr(&s->non_finite, 1u);
        }
    }
}

__global__ void k_stats_final(hcmx_stats* st, uint64_t nbuf) {
    for (uint64_t b = blockIdx.x * blockDim.x + threadIdx.x; b < nbuf; b += gridDim.x * blockDim.x)
        if (st[b].all_zero) {
            st[b].min_mag = 0.0;
            st[b].max_mag = 0.0;
        }
}

// --------------------------------------------------------------- pack ----
__device__ __forceinline__ uint64_t encode_value(double v, unsigned e, unsigned m, double inv_scale,
                                                 uint64_t max_offset, uint64_t round_add,
                                                 uint64_t mant_mask) {
    const uint64_t sign = dbits(v) >> 63;
    uint64_t field = sign << (e + m);
    if (v != 0.0) {
        const double vp = __dadd_rn(__dmul_rn(fabs(v), inv_scale), 1.0);  // >= 2, no FMA
        const uint64_t u = dbits(vp) + round_add;
        uint64_t offset = (u >> 52) - 1023;
        uint64_t mant = (u >> (52 - m)) & mant_mask;
        if (offset > max_offset || !isfinite(vp)) {
            offset = max_offset;
            mant = (1ull << m) - 1;
        }
        field |= (offset << m) | mant;
    }
    return field;
}

// Packing without atomics: lane j encodes value 32g + j into a 64-bit field F_j;
// lane K then assembles output word K of the group (bits [32K, 32K+32)) from
// the <= ceil(32/w)+1 fields that overlap it, fetched with warp shuffles.  The
// w words of a group are stored by w lanes at once (coalesced).  Groups
// [g0, g1) of the buffer v[0, n) are packed into out (word 0 = group 0).
__device__ __forceinline__ int pack_groups(const double* __restrict__ v, uint64_t n, uint32_t g0, uint32_t g1,
                                           unsigned e, unsigned m, unsigned w, double scale,
                                           uint32_t* __restrict__ out, unsigned lane, uint32_t gstride = 1) {
    const double inv_scale = 1.0 / scale;  // IEEE division (codec.cpp:107)
    const uint64_t max_offset = (1ull << e) - 1;
    const uint64_t round_add = (m < 52) ? (1ull << (51 - m)) : 0;
    const uint64_t mant_mask = (m == 52) ? ((1ull << 52) - 1) : ((1ull << m) - 1);
    const unsigned T = (32 + w - 1) / w + 1;  // fields overlapping one output word
    const unsigned i0a = (32 * lane) / w, i0b = (32 * (lane + 32)) / w;
    int nf_bad = 0;
    for (uint32_t g4 = g0; g4 < g1; g4 += 4 * gstride) {
        double xs[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t g = g4 + i * gstride;
            const uint64_t idx = (uint64_t)g * 32 + lane;
            xs[i] = (g < g1 && idx < n) ? __ldcs(v + idx) : 0.0;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t g = g4 + i * gstride;
            if (g >= g1) break;
            const uint64_t idx = (uint64_t)g * 32 + lane;
            uint64_t f = 0;
            if (idx < n) {
                if (!isfinite(xs[i])) nf_bad = 1;
                else f = encode_value(xs[i], e, m, inv_scale, max_offset, round_add, mant_mask);
            }
            const uint32_t flo = static_cast<uint32_t>(f), fhi = static_cast<uint32_t>(f >> 32);
            const uint64_t nvalid = umin64(32, n - (uint64_t)g * 32);
            const unsigned nwords = (unsigned)((nvalid * w + 31) / 32);
            uint32_t* o = out + (uint64_t)g * w;
            for (unsigned half = 0; half < (w > 32 ? 2u : 1u); ++half) {
                const unsigned K = lane + 32 * half;
                const unsigned i0 = half ? i0b : i0a;
                uint32_t word = 0;
                for (unsigned t = 0; t < T; ++t) {
                    const unsigned i = i0 + t;
                    const uint32_t lo = __shfl_sync(0xffffffffu, flo, i & 31u);
                    const uint32_t hi = __shfl_sync(0xffffffffu, fhi, i & 31u);
                    const int sft = static_cast<int>(i * w) - static_cast<int>(32 * K);
                    if (i < 32 && sft < 32) {
                        const uint64_t F = (static_cast<uint64_t>(hi) << 32) | lo;
                        word |= sft >= 0 ? static_cast<uint32_t>(F << sft) : static_cast<uint32_t>(F >> (-sft));
                    }
                }
                if (K < nwords) __stcs(o + K, word);
            }
        }
    }
    return __any_sync(0xffffffffu, nf_bad);
}

// Packing of 32-bit fields (w <= 32): lane j encodes value 32g + j into field
// f at bit j w of the group; its low part goes to word q = j w / 32, its high
// part (if it straddles) to word q + 1, ORed into a per-warp shared buffer
// (shared atomics; a word has <= ceil(32 / w) + 1 writers); the w words are
// then stored coalesced.  Four groups share each round of warp barriers.  The
// field arithmetic is encode_value's in 32 bits (e + m <= 31): same bits.
__device__ __forceinline__ int pack_groups32(const double* __restrict__ v, uint32_t n, uint32_t g0, uint32_t g1,
                                             unsigned e, unsigned m, unsigned w, double scale,
                                             uint32_t* __restrict__ out, unsigned lane, uint32_t gstride,
                                             uint32_t* __restrict__ sw) {
    const double inv_scale = 1.0 / scale;  // IEEE division (codec.cpp:107)
    const uint32_t max_offset = (1u << e) - 1u;
    const uint64_t round_add = 1ull << (51 - m);
    const uint32_t mant_mask = (1u << m) - 1u;
    const unsigned sgn_sh = e + m;
    const bool m_lo = m <= 20;
    const unsigned msh = m_lo ? 20u - m : 52u - m;
    const unsigned bit = lane * w, q = bit >> 5, s = bit & 31u;
    const uint32_t nfull = n / 32;
    int nf_bad = 0;
    auto encode = [&](double x) -> uint32_t {
        // the caller rejected non-finite input; zeros keep only their sign
        // (selected, not branched: 1 / scale may be inf for a subnormal scale)
        const uint32_t sign = static_cast<uint32_t>(__double2hiint(x)) >> 31;
        const double vp = __dadd_rn(__dmul_rn(fabs(x), inv_scale), 1.0);  // no FMA (codec.cpp:124)
        const uint64_t u = dbits(vp) + round_add;
        const uint32_t uh = static_cast<uint32_t>(u >> 32), ul = static_cast<uint32_t>(u);
        uint32_t offset = (uh >> 20) - 1023u;
        uint32_t mant = (m_lo ? uh >> msh : __funnelshift_r(ul, uh, msh)) & mant_mask;
        const bool sat = offset > max_offset || static_cast<uint32_t>(__double2hiint(vp)) >= 0x7ff00000u;
        offset = sat ? max_offset : offset;
        mant = sat ? mant_mask : mant;
        return (sign << sgn_sh) | (x != 0.0 ? (offset << m) | mant : 0u);
    };
    for (uint32_t g4 = g0; g4 < g1; g4 += 4 * gstride) {
        // four whole groups (warp-uniform): no bounds on loads or stores
        const bool whole = g4 + 3 * gstride < nfull;
        double xs[4];
        if (whole) {
            const double* vp = v + g4 * 32 + lane;
#pragma unroll
            for (int i = 0; i < 4; ++i) xs[i] = __ldcs(vp + i * gstride * 32);
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t g = g4 + i * gstride;
                const uint32_t idx = g * 32 + lane;
                xs[i] = (g < g1 && idx < n) ? __ldcs(v + idx) : 0.0;
            }
        }
        uint32_t f[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            f[i] = encode(xs[i]);
            sw[i * 36 + lane] = 0u;
            if (lane == 0) sw[i * 36 + 32] = 0u;
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            // the high part is 0 when the field does not straddle (ORing 0 into
            // word q + 1 <= 32 is harmless): no divergent branch
            atomicOr(sw + i * 36 + q, f[i] << s);
            atomicOr(sw + i * 36 + q + 1, __funnelshift_l(f[i], 0u, s));
        }
        __syncwarp();
        if (whole) {
            if (lane < w) {
                uint32_t* op = out + g4 * w + lane;
#pragma unroll
                for (int i = 0; i < 4; ++i) __stcs(op + i * gstride * w, sw[i * 36 + lane]);
            }
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t g = g4 + i * gstride;
                if (g >= g1) break;
                const unsigned nwords = g < nfull ? w : ((n - g * 32) * w + 31) / 32;
                if (lane < nwords) __stcs(out + g * w + lane, sw[i * 36 + lane]);
            }
        }
        __syncwarp();
    }
    return __any_sync(0xffffffffu, nf_bad);
}

__global__ void __launch_bounds__(kWarpsPerBlock * 32)
k_pack(const double* __restrict__ values, const uint64_t* __restrict__ voff,
       const uint64_t* __restrict__ count, const hcmx_descriptor* __restrict__ desc,
       const uint64_t* __restrict__ poff, const Job* __restrict__ jobs, uint64_t njobs,
       uint8_t* __restrict__ payload, int* __restrict__ err) {
    const unsigned lane = threadIdx.x & 31;
    const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    for (uint64_t j = wid; j < njobs; j += nw) {
        const Job jb = jobs[j];
        const hcmx_descriptor d = desc[jb.buf];
        const int bad = pack_groups(values + voff[jb.buf], count[jb.buf], jb.g0, jb.g0 + jb.ng, d.exp_bits,
                                    d.mant_bits, d.bit_width, d.scale,
                                    reinterpret_cast<uint32_t*>(payload + poff[jb.buf]), lane);
        if (bad && lane == 0) *err = 1;
    }
}

// The layout of one buffer from its reduced statistics (codec.cpp:62-101 with
// the device log2; `ambiguous` flags an exponent width the host must re-decide
// with glibc, see k_compress_cta), written by thread 0 as descriptor, stats and
// flags.  Returns w, e, m and the scale through the references.
__device__ __forceinline__ void cta_layout(uint64_t b, uint64_t mn, uint64_t mx, unsigned nz, unsigned nf, int scheme,
                                           unsigned m_req, unsigned tid, hcmx_descriptor* __restrict__ desc,
                                           hcmx_stats* __restrict__ stats, uint32_t* __restrict__ flags,
                                           unsigned& e_out, unsigned& m_out, unsigned& w_out, double& scale_out) {
    const bool all_zero = !nz;
    const double dmin = all_zero ? 0.0 : bitsd(mn), dmax = all_zero ? 0.0 : bitsd(mx);
    unsigned e = 2, ambiguous = 0;
    if (scheme == HCMX_BFL) {
        e = 8;
    } else if (scheme == HCMX_DFL) {
        e = 11;
    } else if (!all_zero) {  // codec.cpp:69-75: e = ceil(log2(log2 max - log2 min + 2)), estimated
        // log2 of each magnitude = exact binary exponent + MUFU log2 of the
        // mantissa in [1, 2) (absolute error < 4e-7 each, subnormals through the
        // libdevice log2); a value of vv within 1e-6 (relative) of a power of two
        // 2^2..2^10 -- where the estimate could pick the other width -- is flagged
        // and the host re-decides with glibc log2 exactly like the reference
        auto lg = [](double x) -> double {
            const uint32_t hi = static_cast<uint32_t>(__double2hiint(x));
            const int be = static_cast<int>((hi >> 20) & 0x7ffu);
            if (be == 0) return log2(x);  // subnormal (rare): the libdevice log2
            const double mnt = __hiloint2double(static_cast<int>((hi & 0x000fffffu) | 0x3ff00000u), __double2loint(x));
            return static_cast<double>(be - 1023) + static_cast<double>(__log2f(static_cast<float>(mnt)));
        };
        const double vv = (lg(dmax) - lg(dmin) + 1.0) + 1.0;
        // ceil(log2(vv)) away from powers of two: the exponent of vv, plus 1
        // unless vv = 2^k exactly.  Ambiguous: vv within 2^-16 (relative) of
        // 2^2..2^10, read off the top 20 mantissa bits with integer ops (the
        // estimate's error is < 2e-7 relative)
        const uint32_t vh = static_cast<uint32_t>(__double2hiint(vv)), fr = vh & 0x000fffffu;
        const int ve = static_cast<int>((vh >> 20) & 0x7ffu) - 1023;
        const bool pow2 = fr == 0u && __double2loint(vv) == 0;
        const int bits = pow2 ? ve : ve + 1;
        e = static_cast<unsigned>(min(max(bits, 2), 11));
        ambiguous = ((fr < 16u && ve >= 2 && ve <= 10) || (fr >= 0xffff0u && ve >= 1 && ve <= 9)) ? 1u : 0u;
    }
    unsigned m = m_req;
    const unsigned unit = scheme == HCMX_AFL ? 1u : (scheme == HCMX_DFL ? 16u : 8u);
    if (scheme != HCMX_AFL) {  // codec.cpp:25-30
        unsigned w0 = 1 + e + m;
        w0 += (unit - w0 % unit) % unit;
        m = min(52u, w0 - 1 - e);
    }
    unsigned w = 1 + e + m;
    w += (unit - w % unit) % unit;
    const double scale = all_zero ? 1.0 : dmin;
    if (tid == 0) {
        hcmx_descriptor d;
        d.scheme = static_cast<uint8_t>(scheme);
        d.exp_bits = static_cast<uint8_t>(e);
        d.mant_bits = static_cast<uint8_t>(m);
        d.bit_width = static_cast<uint8_t>(w);
        d.reserved = 0;
        d.scale = scale;
        desc[b] = d;
        hcmx_stats st;
        st.min_mag = dmin;
        st.max_mag = dmax;
        st.all_zero = all_zero ? 1u : 0u;
        st.non_finite = nf;
        if (stats) stats[b] = st;
        flags[b] = ambiguous | (nf ? 2u : 0u);  // bit 1: non-finite input (rejected)
    }
    e_out = e;
    m_out = m;
    w_out = w;
    scale_out = scale;
}

// codec.cpp:142-144 fused per buffer, one CTA of kCtaWarps warps per buffer:
// pass 1 (min/max, every thread, 8 loads in flight), block reduction, the
// layout rules, pass 2 packs groups warp-strided (the values come back from
// L2).  The exponent width uses the device log2; when log2(max) - log2(min) + 2
// falls within 1e-9 (relative) of a power of two 2^2..2^10 the buffer is
// flagged and the host re-decides with glibc's log2 exactly like the reference
// (and repacks if it differs).
constexpr int kCtaWarps = 4;

__global__ void __launch_bounds__(kCtaWarps * 32)
k_compress_cta(const double* __restrict__ values, const uint64_t* __restrict__ voff,
               const uint64_t* __restrict__ count, uint64_t nbuf, int scheme, unsigned m_req,
               const uint64_t* __restrict__ poff, uint8_t* __restrict__ payload,
               hcmx_descriptor* __restrict__ desc, hcmx_stats* __restrict__ stats,
               uint32_t* __restrict__ flags) {
    __shared__ uint64_t s_mn[kCtaWarps], s_mx[kCtaWarps];
    __shared__ unsigned s_nz[kCtaWarps], s_nf[kCtaWarps];
    __shared__ uint32_t s_words[kCtaWarps][4][36];
    const unsigned tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    for (uint64_t b = blockIdx.x; b < nbuf; b += gridDim.x) {
        const uint64_t n = count[b];  // <= kFuseMax
        const uint32_t n32 = static_cast<uint32_t>(n);
        const double* v = values + voff[b];
        // min / max of the nonzero |v| on the bit patterns (non-negative doubles
        // order like their bits).  |v| - 1 wraps a zero to the largest value, so
        // the min skips zeros without a test; a non-finite value shows up as a
        // max at or above +inf (the buffer is then rejected, codec.cpp:119-120).
        uint64_t mnm1 = ~0ull, mx = 0;
        uint32_t orv = 0;
        constexpr unsigned T = kCtaWarps * 32;
        for (uint32_t i = tid; i < n32; i += 8 * T) {
            uint64_t xs[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                xs[u] = i + T * u < n32 ? static_cast<uint64_t>(__ldcg(reinterpret_cast<const long long*>(v) + i + T * u))
                                        : 0ull;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint64_t a = xs[u] & 0x7fffffffffffffffull;
                orv |= static_cast<uint32_t>(a >> 32) | static_cast<uint32_t>(a);
                const uint64_t am1 = a - 1;
                mnm1 = am1 < mnm1 ? am1 : mnm1;
                mx = a > mx ? a : mx;
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const uint64_t omn = __shfl_xor_sync(0xffffffffu, mnm1, o);
            const uint64_t omx = __shfl_xor_sync(0xffffffffu, mx, o);
            mnm1 = omn < mnm1 ? omn : mnm1;
            mx = omx > mx ? omx : mx;
        }
        unsigned nz = __any_sync(0xffffffffu, orv != 0);
        unsigned nf = mx >= 0x7FF0000000000000ull ? 1u : 0u;
        if (lane == 0) {
            s_mn[warp] = mnm1;
            s_mx[warp] = mx;
            s_nz[warp] = nz;
            s_nf[warp] = nf;
        }
        __syncthreads();
        mnm1 = s_mn[0];
        mx = s_mx[0];
        nz = s_nz[0];
        nf = s_nf[0];
#pragma unroll
        for (int q = 1; q < kCtaWarps; ++q) {
            mnm1 = s_mn[q] < mnm1 ? s_mn[q] : mnm1;
            mx = s_mx[q] > mx ? s_mx[q] : mx;
            nz |= s_nz[q];
            nf |= s_nf[q];
        }
        const uint64_t mn = mnm1 + 1;
        __syncthreads();  // s_* reused by the next buffer
        unsigned e, m, w;
        double scale;
        cta_layout(b, mn, mx, nz, nf, scheme, m_req, tid, desc, stats, flags, e, m, w, scale);
        if (nf) continue;
        if (w <= 32)
            pack_groups32(v, n32, warp, (n32 + 31) / 32, e, m, w, scale,
                          reinterpret_cast<uint32_t*>(payload + poff[b]), lane, kCtaWarps, &s_words[warp][0][0]);
        else
            pack_groups(v, n, warp, static_cast<uint32_t>((n + 31) / 32), e, m, w, scale,
                        reinterpret_cast<uint32_t*>(payload + poff[b]), lane, kCtaWarps);
    }
}

// The same for buffers of <= kRegMax values (config 2's 64 x 64 blocks): one
// CTA of kCtaWarps warps per buffer, every value loaded exactly once into
// registers (lane l of warp q holds values 32 g + l of groups g = q, q + 4, ...,
// all loads in flight together), the statistics reduced from the registers,
// then encoded and packed from the same registers (no second pass over HBM or
// L2).  Grid: the resident CTAs of the device, buffers strided over them.
constexpr int kRegJ = 32;                                  // values per thread
constexpr uint64_t kRegMax = uint64_t(kRegJ) * kCtaWarps * 32;  // 4096

template <bool ZSEL = true>
__device__ __forceinline__ uint32_t encode32(double x, double inv_scale, uint64_t round_add, bool m_lo, unsigned msh,
                                             uint32_t mant_mask, uint32_t max_offset, unsigned sgn_sh, unsigned m) {
    // the field arithmetic of encode_value in 32 bits.  Zeros keep only their
    // sign: with a finite 1 / scale a zero already encodes to offset 0, mantissa
    // 0 (vp = 1.0 exactly), so the select is needed (ZSEL) only when 1 / scale
    // is infinite (a subnormal scale: 0 * inf is NaN)
    const uint32_t sign = static_cast<uint32_t>(__double2hiint(x)) >> 31;
    const double vp = __dadd_rn(__dmul_rn(fabs(x), inv_scale), 1.0);  // no FMA (codec.cpp:124)
    const uint64_t u = dbits(vp) + round_add;
    const uint32_t uh = static_cast<uint32_t>(u >> 32), ul = static_cast<uint32_t>(u);
    uint32_t offset = (uh >> 20) - 1023u;
    uint32_t mant = (m_lo ? uh >> msh : __funnelshift_r(ul, uh, msh)) & mant_mask;
    const bool sat = offset > max_offset || static_cast<uint32_t>(__double2hiint(vp)) >= 0x7ff00000u;
    offset = sat ? max_offset : offset;
    mant = sat ? mant_mask : mant;
    if (ZSEL) return (sign << sgn_sh) | (x != 0.0 ? (offset << m) | mant : 0u);
    return (sign << sgn_sh) | (offset << m) | mant;
}

__global__ void __launch_bounds__(kCtaWarps * 32, HCMX_REG_MINB)
k_compress_reg(const double* __restrict__ values, const uint64_t* __restrict__ voff,
               const uint64_t* __restrict__ count, uint64_t nbuf, int scheme, unsigned m_req,
               const uint64_t* __restrict__ poff, uint8_t* __restrict__ payload,
               hcmx_descriptor* __restrict__ desc, hcmx_stats* __restrict__ stats,
               uint32_t* __restrict__ flags) {
    __shared__ uint64_t s_mn[kCtaWarps], s_mx[kCtaWarps];
    __shared__ unsigned s_nz[kCtaWarps], s_nf[kCtaWarps];
    __shared__ uint32_t s_words[kCtaWarps][4][36];
    const unsigned tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    uint32_t* sw = &s_words[warp][0][0];
    for (uint64_t b = blockIdx.x; b < nbuf; b += gridDim.x) {
        const uint32_t n = static_cast<uint32_t>(count[b]);  // <= kRegMax
        const double* v = values + voff[b];
        const uint32_t ngroups = (n + 31) / 32, nfull = n / 32;
        double xs[kRegJ];
        if (n == kRegMax) {
#pragma unroll
            for (int j = 0; j < kRegJ; ++j) xs[j] = __ldcs(v + (warp + kCtaWarps * j) * 32 + lane);
        } else {
#pragma unroll
            for (int j = 0; j < kRegJ; ++j) {
                const uint32_t idx = (warp + kCtaWarps * j) * 32 + lane;
                xs[j] = idx < n ? __ldcs(v + idx) : 0.0;
            }
        }
        uint64_t mnm1 = ~0ull, mx = 0;
        uint32_t orv = 0;
#pragma unroll
        for (int j = 0; j < kRegJ; ++j) {
            const uint64_t a = dbits(xs[j]) & 0x7fffffffffffffffull;
            orv |= static_cast<uint32_t>(a >> 32) | static_cast<uint32_t>(a);
            const uint64_t am1 = a - 1;
            mnm1 = am1 < mnm1 ? am1 : mnm1;
            mx = a > mx ? a : mx;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const uint64_t omn = __shfl_xor_sync(0xffffffffu, mnm1, o);
            const uint64_t omx = __shfl_xor_sync(0xffffffffu, mx, o);
            mnm1 = omn < mnm1 ? omn : mnm1;
            mx = omx > mx ? omx : mx;
        }
        unsigned nz = __any_sync(0xffffffffu, orv != 0);
        unsigned nf = mx >= 0x7FF0000000000000ull ? 1u : 0u;
        if (lane == 0) {
            s_mn[warp] = mnm1;
            s_mx[warp] = mx;
            s_nz[warp] = nz;
            s_nf[warp] = nf;
        }
        __syncthreads();
        mnm1 = s_mn[0];
        mx = s_mx[0];
        nz = s_nz[0];
        nf = s_nf[0];
#pragma unroll
        for (int q = 1; q < kCtaWarps; ++q) {
            mnm1 = s_mn[q] < mnm1 ? s_mn[q] : mnm1;
            mx = s_mx[q] > mx ? s_mx[q] : mx;
            nz |= s_nz[q];
            nf |= s_nf[q];
        }
        __syncthreads();  // s_* reused by the next buffer
        unsigned e, m, w;
        double scale;
        cta_layout(b, mnm1 + 1, mx, nz, nf, scheme, m_req, tid, desc, stats, flags, e, m, w, scale);
        if (nf) continue;
        uint32_t* out = reinterpret_cast<uint32_t*>(payload + poff[b]);
        if (w > 32) {  // 64-bit fields: the streaming packer (values come back from L2)
            pack_groups(v, n, warp, ngroups, e, m, w, scale, out, lane, kCtaWarps);
            continue;
        }
        const double inv_scale = 1.0 / scale;  // IEEE division (codec.cpp:107)
        const uint32_t max_offset = (1u << e) - 1u;
        const uint64_t round_add = 1ull << (51 - m);
        const uint32_t mant_mask = (1u << m) - 1u;
        const bool m_lo = m <= 20;
        const unsigned msh = m_lo ? 20u - m : 52u - m;
        const unsigned bit = lane * w, q = bit >> 5, sh = bit & 31u;
#pragma unroll
        for (int j4 = 0; j4 < kRegJ; j4 += 4) {
            const uint32_t gb = warp + kCtaWarps * j4;  // group of round element 0
            if (gb >= ngroups) break;
            uint32_t f[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                f[i] = encode32(xs[j4 + i], inv_scale, round_add, m_lo, msh, mant_mask, max_offset, e + m, m);
                sw[i * 36 + lane] = 0u;
                if (lane == 0) sw[i * 36 + 32] = 0u;
            }
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                // zeros past n encode to 0 (ORing them is harmless)
                atomicOr(sw + i * 36 + q, f[i] << sh);
                atomicOr(sw + i * 36 + q + 1, __funnelshift_l(f[i], 0u, sh));
            }
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t g = gb + kCtaWarps * i;
                if (g < nfull) {
                    if (lane < w) __stcs(out + g * w + lane, sw[i * 36 + lane]);
                } else if (g < ngroups) {
                    const unsigned nwords = ((n - g * 32) * w + 31) / 32;
                    if (lane < nwords) __stcs(out + g * w + lane, sw[i * 36 + lane]);
                }
            }
            __syncwarp();
        }
    }
}

// The same for buffers of <= kRegMax values, with the buffer staged in shared
// memory by one bulk copy (TMA engine) into a 2-slot ring: the copy of the
// CTA's next buffer is in flight while the current one is analysed, encoded
// and packed from shared memory, so the CTA never waits on HBM after its first
// buffer.  Per buffer: statistics (every warp) | barrier | layout (warp 0:
// exponent-width estimate, 1 / scale, descriptor) | barrier | encode + pack.
// Buffers whose values are not 16-byte aligned are copied by the threads
// instead (same results).  (Measured and rejected: register-resident values,
// 4 / 16 warps, a 3-slot ring with the layout overlapped by the next buffer's
// statistics -- 2 CTAs per SM instead of 3 lose more than the overlap gains.)
#ifndef HCMX_TMA_WARPS
#define HCMX_TMA_WARPS 8
#endif
constexpr int kTmaWarps = HCMX_TMA_WARPS;
constexpr uint32_t kTmaSlotBytes = static_cast<uint32_t>(kRegMax) * 8;  // 32 KB
constexpr size_t kTmaSmem = 2 * size_t(kTmaSlotBytes) + 16;               // 2 slots + 2 mbarriers

__device__ __forceinline__ uint32_t cx_smem(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ bool cx_try_wait(uint64_t* bar, unsigned parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 1000;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(cx_smem(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// 64-bit unsigned min / max over the warp with the 32-bit REDUX unit: the
// high words first, then the low words of the lanes holding that high word
__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
    const uint32_t hi = static_cast<uint32_t>(v >> 32), lo = static_cast<uint32_t>(v);
    const uint32_t mh = __reduce_min_sync(0xffffffffu, hi);
    const uint32_t ml = __reduce_min_sync(0xffffffffu, hi == mh ? lo : 0xffffffffu);
    return (static_cast<uint64_t>(mh) << 32) | ml;
}
__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
    const uint32_t hi = static_cast<uint32_t>(v >> 32), lo = static_cast<uint32_t>(v);
    const uint32_t mh = __reduce_max_sync(0xffffffffu, hi);
    const uint32_t ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
    return (static_cast<uint64_t>(mh) << 32) | ml;
}

__global__ void __launch_bounds__(kTmaWarps * 32)
k_compress_tma(const double* __restrict__ values, const uint64_t* __restrict__ voff,
               const uint64_t* __restrict__ count, uint64_t nbuf, int scheme, unsigned m_req,
               const uint64_t* __restrict__ poff, uint8_t* __restrict__ payload,
               hcmx_descriptor* __restrict__ desc, hcmx_stats* __restrict__ stats,
               uint32_t* __restrict__ flags) {
    extern __shared__ __align__(128) uint8_t cx_smem_buf[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(cx_smem_buf + 2 * kTmaSlotBytes);
    __shared__ uint64_t s_mn[kTmaWarps], s_mx[kTmaWarps];
    __shared__ unsigned s_nz[kTmaWarps], s_nf[kTmaWarps], s_manual[2];
    __shared__ struct {
        unsigned e, m, w, nf;
        double scale, inv;
    } s_par;
    __shared__ __align__(16) uint32_t s_words[kTmaWarps][4 * 32 + 4];
    const unsigned tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    constexpr unsigned T = kTmaWarps * 32;
    uint32_t* sw = &s_words[warp][0];
    for (unsigned i = lane; i < 4 * 32 + 4; i += 32) sw[i] = 0u;  // kept zero between rounds (read-and-clear)
    if (tid == 0) {
        for (int i = 0; i < 2; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(cx_smem(bar + i)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // thread 0: start the copy of a buffer of n values at src into slot sl (or
    // flag it for a thread copy)
    auto issue = [&](uint64_t n, const double* src, unsigned sl) {
        const unsigned bytes = static_cast<unsigned>(n * 8);
        const bool bulk = ((reinterpret_cast<uintptr_t>(src) | bytes) & 15u) == 0 && bytes;
        s_manual[sl] = bulk ? 0u : 1u;
        const uint32_t bs = cx_smem(bar + sl);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bs), "r"(bulk ? bytes : 0u)
                     : "memory");
        if (bulk)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    cx_smem(cx_smem_buf + sl * kTmaSlotBytes)),
                "l"(src), "r"(bytes), "r"(bs)
                : "memory");
    };
    uint64_t b = blockIdx.x;
    if (b < nbuf && tid == 0) issue(count[b], values + voff[b], 0);
    for (uint32_t it = 0; b < nbuf; ++it, b += gridDim.x) {
        const unsigned sl = it & 1u, par = (it >> 1) & 1u;
        // the index loads this iteration needs later, issued before the waits
        // (no dependent global load on the path after a barrier)
        const uint32_t n = static_cast<uint32_t>(count[b]);  // <= kRegMax
        uint32_t* out = reinterpret_cast<uint32_t*>(payload + poff[b]);
        const bool has_next = b + gridDim.x < nbuf;
        uint64_t nx_n = 0;
        const double* nx_src = values;
        if (tid == 0 && has_next) {
            nx_n = count[b + gridDim.x];
            nx_src = values + voff[b + gridDim.x];
        }
        while (!cx_try_wait(bar + sl, par)) {
        }
        double* xs = reinterpret_cast<double*>(cx_smem_buf + sl * kTmaSlotBytes);
        if (s_manual[sl]) {  // unaligned source: the threads copy it
            const double* v = values + voff[b];
            for (uint32_t i = tid; i < n; i += T) xs[i] = __ldcs(v + i);
            __syncthreads();
        }
        uint64_t mnm1 = ~0ull, mx = 0;
        uint32_t orv = 0;
        for (uint32_t i = tid; i < n; i += T) {
            const uint64_t a = dbits(xs[i]) & 0x7fffffffffffffffull;
            orv |= static_cast<uint32_t>(a >> 32) | static_cast<uint32_t>(a);
            const uint64_t am1 = a - 1;
            mnm1 = am1 < mnm1 ? am1 : mnm1;
            mx = a > mx ? a : mx;
        }
        mnm1 = warp_min_u64(mnm1);
        mx = warp_max_u64(mx);
        unsigned nz = __any_sync(0xffffffffu, orv != 0);
        unsigned nf = mx >= 0x7FF0000000000000ull ? 1u : 0u;
        if (lane == 0) {
            s_mn[warp] = mnm1;
            s_mx[warp] = mx;
            s_nz[warp] = nz;
            s_nf[warp] = nf;
        }
        __syncthreads();
        // every thread is past iteration it - 1 (it reached this barrier): slot
        // sl ^ 1 is free, start the copy of the CTA's next buffer into it
        if (tid == 0 && has_next) issue(nx_n, nx_src, sl ^ 1u);
        __syncwarp();  // warp 0 reconverged before its shuffles
        if (warp == 0) {  // the layout once per buffer (one warp), broadcast through shared memory
            // the warps' partial statistics: a shuffle tree over lanes 0..kTmaWarps-1
            const unsigned q = lane < kTmaWarps ? lane : 0u;
            mnm1 = warp_min_u64(s_mn[q]);
            mx = warp_max_u64(s_mx[q]);
            nz = __reduce_or_sync(0xffffffffu, s_nz[q]);
            nf = __reduce_or_sync(0xffffffffu, s_nf[q]);
            // 1 / scale first: its Newton chain overlaps the width selection
            const double inv = 1.0 / (nz ? bitsd(mnm1 + 1) : 1.0);  // IEEE division (codec.cpp:107)
            unsigned e, m, w;
            double scale;
            cta_layout(b, mnm1 + 1, mx, nz, nf, scheme, m_req, tid, desc, stats, flags, e, m, w, scale);
            if (lane == 0) {
                s_par.e = e;
                s_par.m = m;
                s_par.w = w;
                s_par.nf = nf;
                s_par.scale = scale;
                s_par.inv = inv;
            }
        }
        __syncthreads();
        const unsigned e = s_par.e, m = s_par.m, w = s_par.w;
        const double scale = s_par.scale;
        if (s_par.nf) continue;
        const uint32_t ngroups = (n + 31) / 32, nfull = n / 32;
        if (w > 32) {  // 64-bit fields: the streaming packer (values re-read from global memory)
            pack_groups(values + voff[b], n, warp, ngroups, e, m, w, scale, out, lane, kTmaWarps);
            continue;
        }
        const double inv_scale = s_par.inv;
        const uint32_t max_offset = (1u << e) - 1u;
        const uint64_t round_add = 1ull << (51 - m);
        const uint32_t mant_mask = (1u << m) - 1u;
        const bool m_lo = m <= 20;
        const unsigned msh = m_lo ? 20u - m : 52u - m;
        const unsigned bit = lane * w, q = bit >> 5, sh = bit & 31u;
        const bool vec_ok = (reinterpret_cast<uintptr_t>(out) & 15u) == 0;
        // Z: zeros need the select (1 / scale infinite); HI: m <= 19, the
        // rounding increment 2^(51 - m) lies in the high word (no carry from the
        // low word), so the field comes from the high word alone
        auto pack = [&](auto zsel, auto hisel) {
            constexpr bool Z = decltype(zsel)::value, HI = decltype(hisel)::value;
            const uint32_t radd_hi = HI ? (1u << (19 - m)) : 0u;
            auto enc = [&](double x) -> uint32_t {
                if (!HI) return encode32<Z>(x, inv_scale, round_add, m_lo, msh, mant_mask, max_offset, e + m, m);
                const uint32_t sign = static_cast<uint32_t>(__double2hiint(x)) >> 31;
                const double vp = __dadd_rn(__dmul_rn(fabs(x), inv_scale), 1.0);  // no FMA (codec.cpp:124)
                const uint32_t uh = static_cast<uint32_t>(__double2hiint(vp)) + radd_hi;
                uint32_t offset = (uh >> 20) - 1023u;
                uint32_t mant = (uh >> msh) & mant_mask;
                const bool sat = offset > max_offset || static_cast<uint32_t>(__double2hiint(vp)) >= 0x7ff00000u;
                offset = sat ? max_offset : offset;
                mant = sat ? mant_mask : mant;
                if (Z) return (sign << (e + m)) | (x != 0.0 ? (offset << m) | mant : 0u);
                return (sign << (e + m)) | (offset << m) | mant;
            };
            // a round: four ADJACENT groups 4j..4j+3 (their 4w packed words are
            // contiguous in the output, 16-byte aligned), packed into the warp's
            // word buffer and stored as w 16-byte vectors
            for (uint32_t g4 = 4 * warp; g4 < ngroups; g4 += 4 * kTmaWarps) {
                uint32_t f[4];
                const bool whole = g4 + 3 < nfull;  // four whole groups (warp-uniform)
                if (whole) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) f[i] = enc(xs[(g4 + i) * 32 + lane]);
                } else {
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const uint32_t idx = (g4 + i) * 32 + lane;
                        f[i] = enc(idx < n ? xs[idx] : 0.0);
                    }
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    // words >= 4w only ever receive zero high parts, so the words
                    // a round reads back are the only ones it must clear
                    atomicOr(sw + i * w + q, f[i] << sh);
                    atomicOr(sw + i * w + q + 1, __funnelshift_l(f[i], 0u, sh));
                }
                __syncwarp();
                uint32_t* o = out + g4 * w;
                if (whole && vec_ok) {
                    if (lane < w) {
                        uint4* sv = reinterpret_cast<uint4*>(sw) + lane;
                        const uint4 v4 = *sv;
                        *sv = make_uint4(0u, 0u, 0u, 0u);
                        __stcs(reinterpret_cast<uint4*>(o) + lane, v4);
                    }
                } else {
                    const uint32_t nw = static_cast<uint32_t>(umin64(4ull * w, ((uint64_t)(n - g4 * 32) * w + 31) / 32));
                    for (uint32_t k = lane; k < 4 * w; k += 32) {
                        const uint32_t word = sw[k];
                        sw[k] = 0u;
                        if (k < nw) __stcs(o + k, word);
                    }
                }
                __syncwarp();
            }
        };
        const bool inf = isinf(inv_scale);
        if (m <= 19) {
            if (inf) pack(std::true_type{}, std::true_type{});
            else pack(std::false_type{}, std::true_type{});
        } else {
            if (inf) pack(std::true_type{}, std::false_type{});
            else pack(std::false_type{}, std::false_type{});
        }
    }
}

// ------------------------------------------------------------- unpack ----
__device__ __forceinline__ double decode_field(uint64_t field, unsigned e, unsigned m, double scale) {
    const uint64_t exp_mask = (1ull << e) - 1;
    const uint64_t mant_mask = (m == 52) ? ((1ull << 52) - 1) : ((1ull << m) - 1);
    const uint64_t sign = (field >> (e + m)) & 1u;
    const uint64_t offset = (field >> m) & exp_mask;
    const uint64_t mant = field & mant_mask;
    double v = 0.0;
    if (offset != 0 || mant != 0) {
        const uint64_t biased = umin64(offset + 1023, 2046);  // codec.cpp:165
        v = __dmul_rn(bitsd((biased << 52) | (mant << (52 - m))) - 1.0, scale);
    }
    return sign ? -v : v;
}

// Job-free unpacking: warp chunks of 32 groups (1024 values); chunk c belongs
// to the buffer found by binary search over coff (cumulative chunks per
// buffer).  A piece of a chunk (all of it for w <= 32, half for w > 32) is
// loaded with 16-byte loads into registers, parked in a per-warp shared
// buffer, and decoded from there while the loads of the warp's NEXT piece are
// already in flight (software pipelining: every warp keeps one piece of
// loads outstanding through its decode and store phase); the doubles are
// stored coalesced with streaming stores.
constexpr int kUnpackWarps = 8;
constexpr unsigned kStageWords = 1024;  // per warp: 16 groups at w <= 64, 32 at w <= 32

// per-chunk metadata, loaded one chunk ahead of the prefetched piece
struct ChunkMeta {
    hcmx_descriptor d;
    uint64_t n, poff, voff, c0;
};
__device__ __forceinline__ ChunkMeta chunk_meta(uint64_t c, const uint32_t* cbuf, const uint64_t* coff,
                                                const hcmx_descriptor* desc, const uint64_t* count,
                                                const uint64_t* poff, const uint64_t* voff) {
    const uint32_t b = __ldg(cbuf + c);
    ChunkMeta m;
    m.d = desc[b];
    m.n = count[b];
    m.poff = poff[b];
    m.voff = voff[b];
    m.c0 = __ldg(coff + b);
    return m;
}

// groups [g0, g1) of the piece of chunk c starting at group g0, and its 16-byte vectors
struct Piece {
    uint32_t g0, g1, nvec;
};
__device__ __forceinline__ Piece piece_of(const ChunkMeta& m, uint64_t c, uint32_t g0) {
    const unsigned w = m.d.bit_width;
    const uint64_t ngroups = (m.n + 31) / 32, nwords_all = (m.n * w + 31) / 32;
    const uint32_t gc1 = static_cast<uint32_t>(umin64((c - m.c0) * 32 + 32, ngroups));
    Piece pc;
    pc.g0 = g0;
    pc.g1 = min(g0 + (w > 32 ? 16u : 32u), gc1);
    const uint64_t wb = (uint64_t)g0 * w, we = umin64((uint64_t)pc.g1 * w, nwords_all);
    pc.nvec = static_cast<unsigned>((we - wb + 3) / 4);  // the slot is 16-byte padded
    return pc;
}
__device__ __forceinline__ void piece_load(const uint8_t* payload, const ChunkMeta& m, const Piece& pc,
                                           unsigned lane, uint4 (&r)[8]) {
    const uint4* src = reinterpret_cast<const uint4*>(payload + m.poff) + (uint64_t)pc.g0 * m.d.bit_width / 4;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const unsigned i = lane + 32u * u;
        if (i < pc.nvec) r[u] = __ldcs(src + i);
    }
}

__global__ void __launch_bounds__(kUnpackWarps * 32, HCMX_UNPACK_MINB)
k_unpack_chunks(const uint8_t* __restrict__ payload, const uint64_t* __restrict__ poff,
                const uint64_t* __restrict__ count, const hcmx_descriptor* __restrict__ desc,
                const uint64_t* __restrict__ voff, const uint64_t* __restrict__ coff,
                const uint32_t* __restrict__ cbuf, uint64_t nchunks, double* __restrict__ out) {
    __shared__ __align__(16) uint32_t stage[kUnpackWarps][kStageWords + 8];
    const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    uint32_t* sw = stage[warp];
    const uint64_t gw = blockIdx.x * (uint64_t)kUnpackWarps + warp;
    const uint64_t nw = gridDim.x * (uint64_t)kUnpackWarps;
    if (gw >= nchunks) return;
    // the prefetched piece (chunk pc_c, meta pm, groups pp) and the meta of the chunk after it
    uint64_t pc_c = gw;
    ChunkMeta pm = chunk_meta(gw, cbuf, coff, desc, count, poff, voff), nm{};
    Piece pp = piece_of(pm, gw, static_cast<uint32_t>((gw - pm.c0) * 32));
    uint4 r[8];
    piece_load(payload, pm, pp, lane, r);
    if (gw + nw < nchunks) nm = chunk_meta(gw + nw, cbuf, coff, desc, count, poff, voff);
    for (;;) {
        const ChunkMeta cm = pm;
        const Piece cp = pp;
        const uint64_t c = pc_c;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const unsigned i = lane + 32u * u;
            if (i < cp.nvec) reinterpret_cast<uint4*>(sw)[i] = r[u];
        }
        __syncwarp();
        // issue the next piece's loads before decoding this one
        bool more = true;
        const uint32_t gc1 = static_cast<uint32_t>(umin64((c - cm.c0) * 32 + 32, (cm.n + 31) / 32));
        if (cp.g1 < gc1) {  // second half of a w > 32 chunk
            pp = piece_of(cm, c, cp.g1);
            piece_load(payload, pm, pp, lane, r);
        } else if (c + nw < nchunks) {
            pc_c = c + nw;
            pm = nm;
            pp = piece_of(pm, pc_c, static_cast<uint32_t>((pc_c - pm.c0) * 32));
            piece_load(payload, pm, pp, lane, r);
            if (pc_c + nw < nchunks) nm = chunk_meta(pc_c + nw, cbuf, coff, desc, count, poff, voff);
        } else {
            more = false;
        }
        const hcmx_descriptor d = cm.d;
        const unsigned e = d.exp_bits, m = d.mant_bits, w = d.bit_width;
        const uint64_t n = cm.n;
        double* o = out + cm.voff;
        const uint32_t g0 = cp.g0, g1 = cp.g1;
        const unsigned bit = lane * w, q = bit >> 5, sh = bit & 31u;
        const uint64_t wmask = (w == 64) ? ~0ull : ((1ull << w) - 1);
        if (w <= 32 && e <= 10 && w == 1 + e + m) {
            // 32-bit fields, no 2046 clamp: the double is built with integer ops
            // (exactly the codec's bits - 1.0, one rounding in * scale)
            const uint32_t mask = 0xffffffffu >> (33u - w);
            const bool lo_m = m <= 20;
            const unsigned s1 = lo_m ? 20u - m : m - 20u;
            const uint32_t nfull = static_cast<uint32_t>(umin64(g1, n / 32));
            uint32_t g = g0;
#pragma unroll 4
            for (; g < nfull; ++g) {
                const uint32_t* gp = sw + (g - g0) * w + q;
                const uint32_t t = __funnelshift_r(gp[0], gp[1], sh);
                const uint32_t pay = t & mask;
                const uint32_t hi = (lo_m ? pay << s1 : pay >> s1) + (1023u << 20);
                const uint32_t lo = lo_m ? 0u : pay << (32u - s1);
                const double v = __dmul_rn(__hiloint2double(hi, lo) - 1.0, d.scale);
                const double sv = __hiloint2double(__double2hiint(v) ^ ((t << (32u - w)) & 0x80000000u),
                                                   __double2loint(v));
                __stcs(o + (uint64_t)g * 32 + lane, sv);
            }
            for (; g < g1; ++g) {  // ragged last group
                const uint32_t* gp = sw + (g - g0) * w + q;
                uint64_t win = ((uint64_t)gp[1] << 32 | gp[0]) >> sh;
                const uint64_t idx = (uint64_t)g * 32 + lane;
                if (idx < n) __stcs(o + idx, decode_field(win & wmask, e, m, d.scale));
            }
        } else {
            for (uint32_t g = g0; g < g1; ++g) {
                const uint32_t* gp = sw + (g - g0) * w + q;
                uint64_t win = ((uint64_t)gp[1] << 32 | gp[0]) >> sh;
                if (sh + w > 64) win |= (uint64_t)gp[2] << (64 - sh);
                const uint64_t idx = (uint64_t)g * 32 + lane;
                if (idx < n) __stcs(o + idx, decode_field(win & wmask, e, m, d.scale));
            }
        }
        __syncwarp();
        if (!more) break;
    }
}

// resident blocks of a kernel on the current device (persistent grids: one
// wave, no tail wave), cached per (kernel slot, device)
template <class K>
int resident_grid(int slot, K kernel, int threads, size_t smem) {
    static std::atomic<int> cache[4][64];
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "device");
    std::atomic<int>& c = cache[slot & 3][dev & 63];
    int v = c.load(std::memory_order_relaxed);
    if (v) return v;
    int sms = 0, per = 0;
    check_cuda(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "attr");
    check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, smem), "occupancy");
    v = std::max(1, sms * std::max(1, per));
    c.store(v, std::memory_order_relaxed);
    return v;
}

int grid_for(uint64_t njobs) {
    const uint64_t blocks = (njobs + kWarpsPerBlock - 1) / kWarpsPerBlock;
    return (int)std::max<uint64_t>(1, std::min<uint64_t>(blocks, 148ull * 16));
}

// Device copies of a batch layout (counts, cumulative unpack chunks, payload
// slot offsets), uploaded once per distinct layout: repeated batched calls on
// the same layout do no host-to-device traffic and no synchronisation.
struct LayoutCache {
    std::mutex mu;
    uint64_t nbuf = ~0ull, nchunks = 0;
    std::vector<uint64_t> h_count, h_poff;  // host copies the device arrays were made from
    DevBuf count, coff, cbuf;
    DevBuf poff;
};
LayoutCache g_layout;

// pinned staging for small device-to-host results (descriptors, flags)
struct Pinned {
    std::mutex mu;
    void* p = nullptr;
    size_t bytes = 0;
    void* get(size_t n) {
        if (n > bytes) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            bytes = 0;
            check_cuda(cudaMallocHost(&p, n), "cudaMallocHost");
            bytes = n;
        }
        return p;
    }
};
Pinned g_pinned;

// optional device timing of the batched codec kernels (CUDA events on the
// launching stream), queried through hcmx_gpu_codec_timing
struct CodecTiming {
    std::mutex mu;
    bool on = false;
    double ms[2] = {0, 0};
    uint64_t n[2] = {0, 0};
    std::vector<std::array<cudaEvent_t, 2>> pend[2];
    std::vector<cudaEvent_t> pool;
    cudaEvent_t take() {
        if (pool.empty()) {
            cudaEvent_t e;
            check_cuda(cudaEventCreate(&e), "event");
            return e;
        }
        cudaEvent_t e = pool.back();
        pool.pop_back();
        return e;
    }
    void drain() {
        for (int k = 0; k < 2; ++k) {
            for (auto& pr : pend[k]) {
                float t = 0;
                check_cuda(cudaEventSynchronize(pr[1]), "event");
                check_cuda(cudaEventElapsedTime(&t, pr[0], pr[1]), "event");
                ms[k] += t;
                ++n[k];
                pool.push_back(pr[0]);
                pool.push_back(pr[1]);
            }
            pend[k].clear();
        }
    }
};
CodecTiming g_ct;

// brackets a kernel launch with events when timing is on (kind 0 compress, 1 decompress)
struct KernelTimer {
    int kind;
    cudaStream_t s;
    cudaEvent_t e0 = nullptr;
    KernelTimer(int k, cudaStream_t st) : kind(k), s(st) {
        std::lock_guard<std::mutex> g(g_ct.mu);
        if (!g_ct.on) return;
        e0 = g_ct.take();
        check_cuda(cudaEventRecord(e0, s), "event");
    }
    void stop() {
        if (!e0) return;
        std::lock_guard<std::mutex> g(g_ct.mu);
        cudaEvent_t e1 = g_ct.take();
        check_cuda(cudaEventRecord(e1, s), "event");
        g_ct.pend[kind].push_back({e0, e1});
        e0 = nullptr;
    }
};

}  // namespace

// layout arrays for h_count (caller holds g_layout.mu)
static void layout_arrays(const uint64_t* h_count, uint64_t nbuf, void* stream) {
    if (g_layout.nbuf == nbuf && std::memcmp(g_layout.h_count.data(), h_count, nbuf * 8) == 0) return;
    check_cuda(cudaDeviceSynchronize(), "layout cache");  // kernels may still read the old arrays
    std::vector<uint64_t> coff(nbuf + 1, 0);
    for (uint64_t b = 0; b < nbuf; ++b) coff[b + 1] = coff[b] + (h_count[b] + 1023) / 1024;
    std::vector<uint32_t> cbuf(coff[nbuf]);
    for (uint64_t b = 0; b < nbuf; ++b)
        for (uint64_t c = coff[b]; c < coff[b + 1]; ++c) cbuf[c] = static_cast<uint32_t>(b);
    g_layout.count.alloc(std::max<uint64_t>(16, nbuf * 8));
    g_layout.coff.alloc((nbuf + 1) * 8);
    g_layout.cbuf.alloc(std::max<uint64_t>(16, cbuf.size() * 4));
    h2d(g_layout.count.p, h_count, nbuf * 8, stream);
    h2d(g_layout.coff.p, coff.data(), (nbuf + 1) * 8, stream);
    h2d(g_layout.cbuf.p, cbuf.data(), cbuf.size() * 4, stream);
    stream_sync(stream);
    g_layout.nbuf = nbuf;
    g_layout.h_count.assign(h_count, h_count + nbuf);
    g_layout.nchunks = coff[nbuf];
    g_layout.h_poff.clear();
}

static const uint64_t* layout_poff(const uint64_t* h_poff, uint64_t nbuf, void* stream) {
    if (g_layout.h_poff.size() != nbuf || std::memcmp(g_layout.h_poff.data(), h_poff, nbuf * 8) != 0) {
        check_cuda(cudaDeviceSynchronize(), "layout cache");
        g_layout.poff.alloc(std::max<uint64_t>(16, nbuf * 8));
        h2d(g_layout.poff.p, h_poff, nbuf * 8, stream);
        stream_sync(stream);
        g_layout.h_poff.assign(h_poff, h_poff + nbuf);
    }
    return g_layout.poff.as<uint64_t>();
}

static void upload_jobs(const std::vector<Job>& jobs, DevBuf& dj, void* stream) {
    dj.alloc(std::max<size_t>(16, jobs.size() * sizeof(Job)));
    h2d(dj.p, jobs.data(), jobs.size() * sizeof(Job), stream);
}

void launch_analyze_jobs(const double* values, const uint64_t* voff, const uint64_t* d_count,
                         const uint64_t* h_count, uint64_t nbuf, hcmx_stats* stats, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const auto jobs = make_jobs(h_count, nbuf);
    DevBuf dj;
    upload_jobs(jobs, dj, stream);
    const int gi = (int)std::min<uint64_t>((nbuf + 255) / 256 + 1, 4096);
    k_stats_init<<<gi, 256, 0, s>>>(stats, nbuf);
    if (!jobs.empty())
        k_analyze<<<grid_for(jobs.size()), kWarpsPerBlock * 32, 0, s>>>(values, voff, d_count,
                                                                         dj.as<Job>(), jobs.size(), stats);
    k_stats_final<<<gi, 256, 0, s>>>(stats, nbuf);
    check_cuda(cudaGetLastError(), "analyze launch");
    stream_sync(stream);  // jobs buffer lifetime
}

// returns nonzero if a non-finite value was met
int launch_pack_jobs(const double* values, const uint64_t* voff, const uint64_t* d_count,
                     const uint64_t* h_count, const hcmx_descriptor* desc, const uint64_t* poff,
                     uint64_t nbuf, uint8_t* payload, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const auto jobs = make_jobs(h_count, nbuf);
    if (jobs.empty()) return 0;
    DevBuf dj, de(sizeof(int));
    upload_jobs(jobs, dj, stream);
    check_cuda(cudaMemsetAsync(de.p, 0, sizeof(int), s), "memset");
    k_pack<<<grid_for(jobs.size()), kWarpsPerBlock * 32, 0, s>>>(values, voff, d_count, desc, poff,
                                                                 dj.as<Job>(), jobs.size(), payload,
                                                                 de.as<int>());
    check_cuda(cudaGetLastError(), "pack launch");
    int err = 0;
    d2h(&err, de.p, sizeof(int), stream);
    stream_sync(stream);
    return err;
}

void launch_unpack_jobs(const uint8_t* payload, const uint64_t* poff, const uint64_t* /*d_count*/,
                        const uint64_t* h_count, const hcmx_descriptor* desc, const uint64_t* voff,
                        uint64_t nbuf, double* out, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    std::lock_guard<std::mutex> g(g_layout.mu);
    layout_arrays(h_count, nbuf, stream);
    const uint64_t nch = g_layout.nchunks;
    if (!nch) return;
    const int grid = (int)std::min<uint64_t>((nch + kUnpackWarps - 1) / kUnpackWarps,
                                             resident_grid(0, k_unpack_chunks, kUnpackWarps * 32, 0));
    KernelTimer kt(1, s);
    k_unpack_chunks<<<grid, kUnpackWarps * 32, 0, s>>>(payload, poff, g_layout.count.as<uint64_t>(), desc, voff,
                                                       g_layout.coff.as<uint64_t>(), g_layout.cbuf.as<uint32_t>(),
                                                       nch, out);
    check_cuda(cudaGetLastError(), "unpack launch");
    kt.stop();
}

// fused compress of buffers of <= kFuseMax values: the register-resident
// kernel when every buffer fits it, else the two-pass CTA kernel; the grid is
// the device's resident CTAs (buffers strided over them, no tail wave)
void launch_compress_fused(const double* values, const uint64_t* voff, const uint64_t* d_count, uint64_t nbuf,
                           uint64_t max_count, int scheme, unsigned m_req, const uint64_t* poff, uint8_t* payload,
                           hcmx_descriptor* desc, hcmx_stats* stats, uint32_t* flags, cudaStream_t s) {
    if (max_count <= kRegMax && HCMX_COMPRESS_KIND == 0) {
        static std::once_flag attr;
        std::call_once(attr, [] {
            check_cuda(cudaFuncSetAttribute(k_compress_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(kTmaSmem)), "attr");
        });
        const int grid = (int)std::min<uint64_t>(nbuf, resident_grid(3, k_compress_tma, kTmaWarps * 32, kTmaSmem));
        k_compress_tma<<<grid, kTmaWarps * 32, kTmaSmem, s>>>(values, voff, d_count, nbuf, scheme, m_req, poff,
                                                              payload, desc, stats, flags);
    } else if (max_count <= kRegMax && HCMX_COMPRESS_KIND == 1) {
        const int grid = (int)std::min<uint64_t>(nbuf, resident_grid(1, k_compress_reg, kCtaWarps * 32, 0));
        k_compress_reg<<<grid, kCtaWarps * 32, 0, s>>>(values, voff, d_count, nbuf, scheme, m_req, poff, payload,
                                                       desc, stats, flags);
    } else {
        const int grid = (int)std::min<uint64_t>(nbuf, resident_grid(2, k_compress_cta, kCtaWarps * 32, 0));
        k_compress_cta<<<grid, kCtaWarps * 32, 0, s>>>(values, voff, d_count, nbuf, scheme, m_req, poff, payload,
                                                       desc, stats, flags);
    }
}

}  // namespace hcmx_gpu

// ================================================================ C-ABI ====
using namespace hcmx_gpu;

namespace {

DevBuf upload_u64(const uint64_t* h, uint64_t n, void* stream) {
    DevBuf d(std::max<uint64_t>(8, n * 8));
    h2d(d.p, h, n * 8, stream);
    return d;
}

void validate_desc(const hcmx_descriptor& d) {
    if (d.scheme > 3 || d.exp_bits > 11 || d.mant_bits < 1 || d.mant_bits > 52)
        throw invalid_argument("invalid codec descriptor");
    if (d.bit_width != bit_width(d.scheme, d.exp_bits, d.mant_bits))
        throw invalid_argument("descriptor bit_width does not match scheme/e/m");
}

// host side of codec::compress for a batch: stats -> descriptors -> offsets
void select_layouts(const std::vector<hcmx_stats>& st, const uint64_t* h_count, uint64_t nbuf,
                    double eps, int scheme, hcmx_descriptor* h_desc, uint64_t* h_poff,
                    uint64_t* total) {
    mantissa_bits_for(eps);  // eps validation first (codec.cpp:63-64)
    uint64_t off = 0;
    for (uint64_t b = 0; b < nbuf; ++b) {
        if (st[b].non_finite) throw invalid_argument("compress: values must be finite");
        h_desc[b] = make_descriptor(scheme, eps, st[b]);
        h_poff[b] = off;
        off += round16(payload_bytes(h_count[b], h_desc[b].bit_width));
    }
    *total = off;
}

}  // namespace

extern "C" {

int hcmx_gpu_init(int device) {
    return guarded([&] {
        require_device();
        check_cuda(cudaSetDevice(device), "cudaSetDevice");
        cudaDeviceProp p{};
        check_cuda(cudaGetDeviceProperties(&p, device), "cudaGetDeviceProperties");
        if (p.major != 10)
            throw cuda_error("libhcmx_gpu is built for sm_100a (B200); device is sm_" +
                             std::to_string(p.major * 10 + p.minor));
    });
}

int hcmx_gpu_codec_analyze(const double* d_values, const uint64_t* d_voff, const uint64_t* h_count,
                           uint64_t nbuf, hcmx_stats* d_stats, void* stream) {
    return guarded([&] {
        require_device();
        DevBuf dc = upload_u64(h_count, nbuf, stream);
        launch_analyze_jobs(d_values, d_voff, dc.as<uint64_t>(), h_count, nbuf, d_stats, stream);
    });
}

int hcmx_gpu_codec_pack(const double* d_values, const uint64_t* d_voff, const uint64_t* h_count,
                        const hcmx_descriptor* d_desc, const uint64_t* d_poff, uint64_t nbuf,
                        uint8_t* d_payload, void* stream) {
    return guarded([&] {
        require_device();
        DevBuf dc = upload_u64(h_count, nbuf, stream);
        if (launch_pack_jobs(d_values, d_voff, dc.as<uint64_t>(), h_count, d_desc, d_poff, nbuf,
                             d_payload, stream))
            throw invalid_argument("compress: values must be finite");
    });
}

int hcmx_gpu_codec_unpack(const uint8_t* d_payload, const uint64_t* d_poff, const uint64_t* h_count,
                          const hcmx_descriptor* d_desc, const uint64_t* d_voff, uint64_t nbuf,
                          double* d_out, void* stream) {
    return guarded([&] {
        require_device();
        launch_unpack_jobs(d_payload, d_poff, nullptr, h_count, d_desc, d_voff, nbuf, d_out, stream);
    });
}

int hcmx_gpu_codec_compress(const double* d_values, const uint64_t* d_voff, const uint64_t* h_count,
                            uint64_t nbuf, double eps, int scheme, uint8_t* d_payload,
                            uint64_t payload_capacity, hcmx_descriptor* h_desc, uint64_t* h_poff,
                            uint64_t* h_total, void* stream) {
    return guarded([&] {
        require_device();
        alignment_unit(scheme);
        const uint8_t m_req = mantissa_bits_for(eps);  // eps validation first (codec.cpp:63-64)
        uint64_t maxc = 0;
        for (uint64_t b = 0; b < nbuf; ++b) maxc = std::max(maxc, h_count[b]);
        if (maxc > kFuseMax) {  // very large buffers: device analyze, host selection, device pack
            DevBuf dc = upload_u64(h_count, nbuf, stream);
            DevBuf dst(std::max<uint64_t>(24, nbuf * sizeof(hcmx_stats)));
            launch_analyze_jobs(d_values, d_voff, dc.as<uint64_t>(), h_count, nbuf, dst.as<hcmx_stats>(),
                                stream);
            std::vector<hcmx_stats> st(nbuf);
            d2h(st.data(), dst.p, nbuf * sizeof(hcmx_stats), stream);
            stream_sync(stream);
            select_layouts(st, h_count, nbuf, eps, scheme, h_desc, h_poff, h_total);
            if (*h_total > payload_capacity) throw invalid_argument("compress: payload capacity too small");
            DevBuf dd(std::max<uint64_t>(16, nbuf * sizeof(hcmx_descriptor)));
            h2d(dd.p, h_desc, nbuf * sizeof(hcmx_descriptor), stream);
            DevBuf dp = upload_u64(h_poff, nbuf, stream);
            if (launch_pack_jobs(d_values, d_voff, dc.as<uint64_t>(), h_count, dd.as<hcmx_descriptor>(),
                                 dp.as<uint64_t>(), nbuf, d_payload, stream))
                throw invalid_argument("compress: values must be finite");
            return;
        }
        // fused path: slots sized for the widest layout the scheme allows (e = 11)
        const hcmx_descriptor widest = make_descriptor(scheme, eps, 1.0, 11);
        uint64_t off = 0;
        for (uint64_t b = 0; b < nbuf; ++b) {
            h_poff[b] = off;
            off += round16(payload_bytes(h_count[b], widest.bit_width));
        }
        *h_total = off;
        if (off > payload_capacity) throw invalid_argument("compress: payload capacity too small");
        std::lock_guard<std::mutex> g(g_layout.mu);
        layout_arrays(h_count, nbuf, stream);
        const uint64_t* dp = layout_poff(h_poff, nbuf, stream);
        // one device block for descriptors | flags, one pinned block for the read-back
        const size_t o_fl = round16(nbuf * sizeof(hcmx_descriptor)), o_end = o_fl + round16(nbuf * 4);
        DevBuf out(o_end);
        DevBuf dst(std::max<uint64_t>(24, nbuf * sizeof(hcmx_stats)));
        cudaStream_t s = (cudaStream_t)stream;
        uint8_t* ob = out.as<uint8_t>();
        KernelTimer kt(0, s);
        launch_compress_fused(d_values, d_voff, g_layout.count.as<uint64_t>(), nbuf, maxc, scheme, m_req, dp,
                              d_payload, reinterpret_cast<hcmx_descriptor*>(ob), dst.as<hcmx_stats>(),
                              reinterpret_cast<uint32_t*>(ob + o_fl), s);
        check_cuda(cudaGetLastError(), "compress launch");
        kt.stop();
        std::lock_guard<std::mutex> gp(g_pinned.mu);
        uint8_t* hb = static_cast<uint8_t*>(g_pinned.get(o_end));
        d2h(hb, ob, o_fl + nbuf * 4, stream);
        stream_sync(stream);
        std::memcpy(h_desc, hb, nbuf * sizeof(hcmx_descriptor));
        const uint32_t* flags = reinterpret_cast<const uint32_t*>(hb + o_fl);
        for (uint64_t b = 0; b < nbuf; ++b)
            if (flags[b] & 2u) throw invalid_argument("compress: values must be finite");
        // exponent widths next to a 2^k - 2 threshold: decide with glibc (codec.cpp:72-73)
        for (uint64_t b = 0; b < nbuf; ++b) {
            if (!(flags[b] & 1u)) continue;
            hcmx_stats st{};
            d2h(&st, dst.as<hcmx_stats>() + b, sizeof(hcmx_stats), stream);
            uint64_t vo = 0;
            d2h(&vo, d_voff + b, 8, stream);
            stream_sync(stream);
            const hcmx_descriptor exact = make_descriptor(scheme, eps, st);
            if (exact.exp_bits == h_desc[b].exp_bits) continue;
            h_desc[b] = exact;
            DevBuf d1(sizeof(hcmx_descriptor));
            h2d(d1.p, &exact, sizeof(hcmx_descriptor), stream);
            DevBuf dv1 = upload_u64(&vo, 1, stream), dc1 = upload_u64(h_count + b, 1, stream),
                   dp1 = upload_u64(h_poff + b, 1, stream);
            launch_pack_jobs(d_values, dv1.as<uint64_t>(), dc1.as<uint64_t>(), h_count + b,
                             d1.as<hcmx_descriptor>(), dp1.as<uint64_t>(), 1, d_payload, stream);
        }
    });
}

int hcmx_gpu_codec_compress_device(const double* d_values, const uint64_t* d_voff, const uint64_t* d_count,
                                   uint64_t nbuf, uint64_t max_count, double eps, int scheme, const uint64_t* d_poff,
                                   uint8_t* d_payload, hcmx_descriptor* d_desc, uint32_t* d_flags, void* stream) {
    return guarded([&] {
        require_device();
        alignment_unit(scheme);
        const uint8_t m_req = mantissa_bits_for(eps);  // eps validation first (codec.cpp:63-64)
        if (max_count > kFuseMax) throw invalid_argument("compress_device: buffers above 2^17 values take hcmx_gpu_codec_compress");
        if (!nbuf) return;
        cudaStream_t s = (cudaStream_t)stream;
        KernelTimer kt(0, s);
        launch_compress_fused(d_values, d_voff, d_count, nbuf, max_count, scheme, m_req, d_poff, d_payload, d_desc,
                              nullptr, d_flags, s);
        check_cuda(cudaGetLastError(), "compress launch");
        kt.stop();
    });
}

int hcmx_gpu_codec_compress_fixup(const double* d_values, const uint64_t* d_voff, const uint64_t* h_count,
                                  uint64_t nbuf, double eps, int scheme, const uint64_t* h_poff, uint8_t* d_payload,
                                  hcmx_descriptor* d_desc, const uint32_t* d_flags, uint64_t* n_fixed, void* stream) {
    return guarded([&] {
        require_device();
        std::vector<uint32_t> fl(nbuf);
        d2h(fl.data(), d_flags, nbuf * 4, stream);
        stream_sync(stream);
        uint64_t fixed = 0;
        for (uint64_t b = 0; b < nbuf; ++b)
            if (fl[b] & 2u) throw invalid_argument("compress: values must be finite");
        for (uint64_t b = 0; b < nbuf; ++b) {
            if (!(fl[b] & 1u)) continue;
            // exponent width next to a 2^k - 2 threshold: decide with glibc (codec.cpp:72-73)
            uint64_t vo = 0;
            d2h(&vo, d_voff + b, 8, stream);
            stream_sync(stream);
            DevBuf dv1 = upload_u64(&vo, 1, stream), dc1 = upload_u64(h_count + b, 1, stream);
            DevBuf dst(sizeof(hcmx_stats));
            launch_analyze_jobs(d_values, dv1.as<uint64_t>(), dc1.as<uint64_t>(), h_count + b, 1,
                                dst.as<hcmx_stats>(), stream);
            hcmx_stats st{};
            hcmx_descriptor cur{};
            d2h(&st, dst.p, sizeof(st), stream);
            d2h(&cur, d_desc + b, sizeof(cur), stream);
            stream_sync(stream);
            const hcmx_descriptor exact = make_descriptor(scheme, eps, st);
            if (exact.exp_bits == cur.exp_bits) continue;
            if (payload_bytes(h_count[b], exact.bit_width) > payload_bytes(h_count[b], make_descriptor(scheme, eps, 1.0, 11).bit_width))
                throw std::logic_error("compress_fixup: slot too small");
            h2d(d_desc + b, &exact, sizeof(exact), stream);
            DevBuf dp1 = upload_u64(h_poff + b, 1, stream);
            launch_pack_jobs(d_values, dv1.as<uint64_t>(), dc1.as<uint64_t>(), h_count + b, d_desc + b,
                             dp1.as<uint64_t>(), 1, d_payload, stream);
            ++fixed;
        }
        stream_sync(stream);
        if (n_fixed) *n_fixed = fixed;
    });
}

int hcmx_gpu_codec_timing(int enable, double* ms_compress, uint64_t* n_compress, double* ms_decompress,
                          uint64_t* n_decompress) {
    return guarded([&] {
        std::lock_guard<std::mutex> g(g_ct.mu);
        g_ct.drain();
        if (ms_compress) *ms_compress = g_ct.ms[0];
        if (n_compress) *n_compress = g_ct.n[0];
        if (ms_decompress) *ms_decompress = g_ct.ms[1];
        if (n_decompress) *n_decompress = g_ct.n[1];
        if (enable >= 0) {  // enable < 0: query only
            g_ct.on = enable != 0;
            g_ct.ms[0] = g_ct.ms[1] = 0;
            g_ct.n[0] = g_ct.n[1] = 0;
        }
    });
}

int hcmx_gpu_compress(const double* h_values, uint64_t count, double eps, int scheme,
                      hcmx_descriptor* desc, uint8_t* h_payload, uint64_t capacity,
                      uint64_t* payload_len) {
    return guarded([&] {
        require_device();
        alignment_unit(scheme);
        mantissa_bits_for(eps);
        DevBuf dv(std::max<uint64_t>(8, count * 8));
        h2d(dv.p, h_values, count * 8, nullptr);
        const uint64_t zero = 0;
        DevBuf dvo = upload_u64(&zero, 1, nullptr);
        DevBuf dpay(round16(count * 8) + 16);
        uint64_t poff = 0, total = 0;
        int st = hcmx_gpu_codec_compress(dv.as<double>(), dvo.as<uint64_t>(), &count, 1, eps, scheme,
                                         dpay.as<uint8_t>(), dpay.bytes, desc, &poff, &total, nullptr);
        if (st == HCMX_INVALID_ARGUMENT) throw invalid_argument(hcmx_gpu_last_error());
        if (st) throw cuda_error(hcmx_gpu_last_error());
        const uint64_t len = payload_bytes(count, desc->bit_width);
        if (len > capacity) throw invalid_argument("compress: output capacity too small");
        d2h(h_payload, dpay.p, len, nullptr);
        stream_sync(nullptr);
        *payload_len = len;
    });
}

int hcmx_gpu_compress_block(const double* h_values, uint64_t count, const hcmx_descriptor* desc,
                            uint8_t* h_payload, uint64_t capacity, uint64_t* payload_len) {
    return guarded([&] {
        require_device();
        validate_desc(*desc);
        const uint64_t len = payload_bytes(count, desc->bit_width);
        if (len > capacity) throw invalid_argument("compress_block: output capacity too small");
        DevBuf dv(std::max<uint64_t>(8, count * 8));
        h2d(dv.p, h_values, count * 8, nullptr);
        const uint64_t zero = 0;
        DevBuf dvo = upload_u64(&zero, 1, nullptr);
        DevBuf dpo = upload_u64(&zero, 1, nullptr);
        DevBuf dd(sizeof(hcmx_descriptor));
        h2d(dd.p, desc, sizeof(hcmx_descriptor), nullptr);
        DevBuf dpay(round16(len) + 16);
        DevBuf dc = upload_u64(&count, 1, nullptr);
        if (launch_pack_jobs(dv.as<double>(), dvo.as<uint64_t>(), dc.as<uint64_t>(), &count,
                             dd.as<hcmx_descriptor>(), dpo.as<uint64_t>(), 1, dpay.as<uint8_t>(), nullptr))
            throw invalid_argument("compress: values must be finite");
        d2h(h_payload, dpay.p, len, nullptr);
        stream_sync(nullptr);
        *payload_len = len;
    });
}

int hcmx_gpu_decompress_into(const hcmx_descriptor* desc, uint64_t count, const uint8_t* h_payload,
                             uint64_t payload_len, double* h_out) {
    return guarded([&] {
        require_device();
        validate_desc(*desc);
        const uint64_t need = payload_bytes(count, desc->bit_width);
        // BitReader throws when a read passes the end (bitstream.hpp:80-82)
        if (payload_len < need) throw corrupt_buffer("bitstream: payload ends inside a value");
        if (count == 0) return;
        DevBuf dpay(round16(need) + 16);
        h2d(dpay.p, h_payload, need, nullptr);
        const uint64_t zero = 0;
        DevBuf dvo = upload_u64(&zero, 1, nullptr);
        DevBuf dpo = upload_u64(&zero, 1, nullptr);
        DevBuf dd(sizeof(hcmx_descriptor));
        h2d(dd.p, desc, sizeof(hcmx_descriptor), nullptr);
        DevBuf dout(count * 8);
        DevBuf dc = upload_u64(&count, 1, nullptr);
        launch_unpack_jobs(dpay.as<uint8_t>(), dpo.as<uint64_t>(), dc.as<uint64_t>(), &count,
                           dd.as<hcmx_descriptor>(), dvo.as<uint64_t>(), 1, dout.as<double>(), nullptr);
        d2h(h_out, dout.p, count * 8, nullptr);
        stream_sync(nullptr);
    });
}

// mixedprec.cpp:155-187 (aplr_compress) batched over leaves with given factors
int hcmx_gpu_aplr_compress(uint64_t nleaves, const uint64_t* h_rows, const uint64_t* h_cols,
                           const uint64_t* h_k, const double* d_W, const uint64_t* h_woff,
                           const double* d_X, const uint64_t* h_xoff, const double* h_sigma,
                           const uint64_t* h_soff, const uint64_t* h_boff, double eps, int scheme,
                           uint8_t* d_payload, uint64_t payload_capacity, hcmx_descriptor* h_desc,
                           uint64_t* h_poff, uint64_t* h_total, void* stream) {
    return guarded([&] {
        require_device();
        alignment_unit(scheme);
        // column buffers: W columns of all leaves, then X columns of all leaves,
        // analysed in two batches (they live in different device arrays)
        uint64_t nb = 0;
        for (uint64_t j = 0; j < nleaves; ++j) nb = std::max(nb, h_boff[j] + 2 * h_k[j]);
        std::vector<uint64_t> wv, wc, xv, xc, wbuf, xbuf;
        for (uint64_t j = 0; j < nleaves; ++j)
            for (uint64_t i = 0; i < h_k[j]; ++i) {
                wv.push_back(h_woff[j] + i * h_rows[j]);
                wc.push_back(h_rows[j]);
                wbuf.push_back(h_boff[j] + i);
                xv.push_back(h_xoff[j] + i * h_cols[j]);
                xc.push_back(h_cols[j]);
                xbuf.push_back(h_boff[j] + h_k[j] + i);
            }
        const uint64_t ncol = wv.size();
        std::vector<hcmx_stats> sw(ncol), sx(ncol);
        if (ncol) {
            DevBuf dst(ncol * sizeof(hcmx_stats));
            DevBuf dwv = upload_u64(wv.data(), ncol, stream), dwc = upload_u64(wc.data(), ncol, stream);
            launch_analyze_jobs(d_W, dwv.as<uint64_t>(), dwc.as<uint64_t>(), wc.data(), ncol,
                                dst.as<hcmx_stats>(), stream);
            d2h(sw.data(), dst.p, ncol * sizeof(hcmx_stats), stream);
            DevBuf dxv = upload_u64(xv.data(), ncol, stream), dxc = upload_u64(xc.data(), ncol, stream);
            launch_analyze_jobs(d_X, dxv.as<uint64_t>(), dxc.as<uint64_t>(), xc.data(), ncol,
                                dst.as<hcmx_stats>(), stream);
            d2h(sx.data(), dst.p, ncol * sizeof(hcmx_stats), stream);
            stream_sync(stream);
        }
        // host: factor-wide e (mixedprec.cpp:168-169), per-column eps_i (174) and scale (177-184)
        uint64_t c = 0;
        for (uint64_t j = 0; j < nleaves; ++j) {
            const uint64_t k = h_k[j];
            if (k == 0) continue;
            hcmx_stats fw{INFINITY, 0.0, 1u, 0u}, fx{INFINITY, 0.0, 1u, 0u};
            for (uint64_t i = 0; i < k; ++i) {
                for (int side = 0; side < 2; ++side) {
                    const hcmx_stats& s = side ? sx[c + i] : sw[c + i];
                    hcmx_stats& f = side ? fx : fw;
                    if (s.non_finite) throw invalid_argument("compress: values must be finite");
                    if (!s.all_zero) {
                        f.all_zero = 0;
                        f.min_mag = std::min(f.min_mag, s.min_mag);
                        f.max_mag = std::max(f.max_mag, s.max_mag);
                    }
                }
            }
            if (fw.all_zero) fw.min_mag = fw.max_mag = 0.0;
            if (fx.all_zero) fx.min_mag = fx.max_mag = 0.0;
            const uint8_t e_w = exponent_bits_for(fw), e_x = exponent_bits_for(fx);
            const double* sig = h_sigma + h_soff[j];
            const double delta = eps * sig[0];
            for (uint64_t i = 0; i < k; ++i) {
                const double eps_i = std::min(0.5, delta / sig[i]);
                const hcmx_stats& a = sw[c + i];
                const hcmx_stats& b = sx[c + i];
                h_desc[wbuf[c + i]] = make_descriptor(scheme, eps_i, a.all_zero ? 1.0 : a.min_mag, e_w);
                h_desc[xbuf[c + i]] = make_descriptor(scheme, eps_i, b.all_zero ? 1.0 : b.min_mag, e_x);
            }
            c += k;
        }
        // payload offsets in buffer order
        std::vector<uint64_t> cnt(nb, 0);
        for (uint64_t i = 0; i < ncol; ++i) {
            cnt[wbuf[i]] = wc[i];
            cnt[xbuf[i]] = xc[i];
        }
        uint64_t off = 0;
        for (uint64_t b = 0; b < nb; ++b) {
            h_poff[b] = off;
            off += round16(payload_bytes(cnt[b], h_desc[b].bit_width));
        }
        *h_total = off;
        if (off > payload_capacity) throw invalid_argument("aplr_compress: payload capacity too small");
        if (!ncol) return;
        std::vector<hcmx_descriptor> dw(ncol), dx(ncol);
        std::vector<uint64_t> pw(ncol), px(ncol);
        for (uint64_t i = 0; i < ncol; ++i) {
            dw[i] = h_desc[wbuf[i]];
            dx[i] = h_desc[xbuf[i]];
            pw[i] = h_poff[wbuf[i]];
            px[i] = h_poff[xbuf[i]];
        }
        DevBuf ddw(ncol * sizeof(hcmx_descriptor)), ddx(ncol * sizeof(hcmx_descriptor));
        h2d(ddw.p, dw.data(), ncol * sizeof(hcmx_descriptor), stream);
        h2d(ddx.p, dx.data(), ncol * sizeof(hcmx_descriptor), stream);
        DevBuf dpw = upload_u64(pw.data(), ncol, stream), dpx = upload_u64(px.data(), ncol, stream);
        DevBuf dwv = upload_u64(wv.data(), ncol, stream), dwc = upload_u64(wc.data(), ncol, stream);
        DevBuf dxv = upload_u64(xv.data(), ncol, stream), dxc = upload_u64(xc.data(), ncol, stream);
        if (launch_pack_jobs(d_W, dwv.as<uint64_t>(), dwc.as<uint64_t>(), wc.data(), ddw.as<hcmx_descriptor>(),
                             dpw.as<uint64_t>(), ncol, d_payload, stream) ||
            launch_pack_jobs(d_X, dxv.as<uint64_t>(), dxc.as<uint64_t>(), xc.data(), ddx.as<hcmx_descriptor>(),
                             dpx.as<uint64_t>(), ncol, d_payload, stream))
            throw invalid_argument("compress: values must be finite");
    });
}

}  // extern "C"
