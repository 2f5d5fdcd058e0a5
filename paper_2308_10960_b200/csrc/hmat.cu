// hmat.cu -- device-resident compressed H-matrix and the fused
// decompress + matrix-vector product (hmatrix.hpp:126-128).
//
// Layout (built once on the host by hcmx_gpu_hmat_create):
//   The packed codec streams of every leaf are re-tiled, field-for-field and
//   bit-identical, into one HBM arena of 16-byte aligned "stages" (<= 32 KB):
//
//   phase A (lowrank X^T x): item = (APLR leaf, <= 256 consecutive columns of
//     the block, <= 16 rank columns); its data is, for each rank column, the
//     fields of that X column over the column chunk, word aligned.  One warp
//     decodes an item with the 256 x values in registers (8 per lane), reduces
//     per rank column with shuffles, and either writes t_i directly (one chunk)
//     or a partial that the last-arriving warp sums in fixed chunk order.
//   phase B (row-stationary): one CTA owns one row block (<= 64 rows, a row
//     leaf cluster) and streams the "stripe" of everything that writes those
//     rows: dense leaves (column groups of 16 columns, each column's |rows|
//     fields) and the W slices of every APLR leaf covering the block.  Lane l
//     owns rows l and l+32; y is written once per row, no atomics.
//
//   Stages are moved HBM -> shared memory with cp.async.bulk (the TMA bulk
//   engine) into a 3-deep ring guarded by mbarriers, so the SM only spends
//   issue slots on the decode itself: two LDS + a funnel shift per field, a
//   few integer ops to rebuild the FP64 pattern, one DADD and one DFMA.
//
// Numerics: decoded values are bit-identical to codec::decompress_into; the
// multiply by the buffer scale is folded into the coefficients (dense: alpha *
// scale per item, lowrank: alpha * sigma_i * scale_X_i * scale_W_i), so the sum
// differs from the oracle only by FP64 reassociation (||dy||/||y|| ~ 1e-15).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "internal.h"

namespace hcmx_gpu {
namespace {

constexpr int kNW = 8;                // warps per CTA
constexpr int kStageBytes = 32768;    // bytes per stage buffer
constexpr int kNStage = 3;            // ring depth
constexpr int kSlack = 16;            // decode reads up to 2 words past a segment
constexpr int kAChunk = 256;          // X fields per A item (8 per lane)
constexpr int kAGroup = 16;           // rank columns per A item
constexpr int kBDenseGroup = 16;      // dense columns per B item
constexpr int kBLRGroup = 32;         // rank columns per B item
constexpr int kRowBlock = 64;         // rows per phase-B CTA (2 per lane)
constexpr int kAStagesPerStripe = 8;  // phase-A stages per CTA

struct Stage {
    uint64_t byte_off;
    uint32_t bytes;
    uint32_t item0;
    uint32_t nitems;
    uint32_t pad;
};
static_assert(sizeof(Stage) == 24, "Stage layout");

struct BItem {
    uint32_t word_off;  // from the stage start
    uint16_t nseg;      // columns in this item
    uint8_t kind;       // 0 dense, 1 lowrank
    uint8_t e;          // exponent bits (lowrank: factor-wide)
    uint32_t a;         // dense: x index of first column; lowrank: global W column id
    uint32_t b;         // dense: dense-leaf id
};
static_assert(sizeof(BItem) == 16, "BItem layout");

struct AItem {
    uint32_t word_off;
    uint16_t nseg;      // rank columns
    uint16_t nf;        // fields per column (<= kAChunk)
    uint32_t xcol;      // global X column id of the first rank column
    uint32_t xidx;      // x index of field 0
    uint32_t leaf;      // lowrank-leaf id
    uint16_t chunk;     // column-chunk index within the leaf
    uint16_t icol0;     // first rank column within the leaf
};
static_assert(sizeof(AItem) == 24, "AItem layout");

struct LeafA {
    uint32_t colbase;   // global column id of rank column 0
    uint32_t k;
    uint32_t pbase;     // partials base (nchunks > 1)
    uint32_t nitems;    // A items of this leaf
    uint32_t nchunks;
    uint32_t e;         // X exponent bits
};

struct DenseInfo {
    double scale;
    uint8_t w, m, e, pad[5];
};
static_assert(sizeof(DenseInfo) == 16, "DenseInfo layout");

struct Params {
    const uint8_t* arena;
    const Stage* stages;
    const BItem* bitems;
    const AItem* aitems;
    const uint32_t* stripe_a;   // [nstripe_a + 1] stage ranges
    const uint32_t* stripe_b;   // [nblocks + 1]
    const uint32_t* row_first;  // [nblocks]
    const uint32_t* row_count;
    const LeafA* leafa;
    const DenseInfo* dense;
    const uint16_t* colw_wm;    // (w | m << 8) per W column
    const uint16_t* colx_wm;
    const double* coef;         // sigma_i * scale_X_i * scale_W_i
    double* c;                  // alpha * coef * (X^T x)_i, written by phase A
    double* partial;
    unsigned* counter;
    const double* x;
    double* y;
    double alpha, beta;
};

// ----------------------------------------------------------- PTX glue ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// ------------------------------------------------------------- decode ----
// Field at bit offset (q * 32 + sh) of the word stream wp, width w, layout
// [mant m][offset e][sign] (codec.cpp:118-137).  Returns (1.mant * 2^offset) - 1
// (exact: the codec's value divided by scale, codec.cpp:161-169) and the sign.
__device__ __forceinline__ double decode_a(const uint32_t* wp, unsigned q, unsigned sh, unsigned w,
                                           unsigned e, unsigned m, uint64_t& sgn) {
    const uint32_t lo = wp[q], hi = wp[q + 1];
    uint64_t win = ((static_cast<uint64_t>(hi) << 32) | lo) >> sh;
    if (w > 32 && sh + w > 64) win |= static_cast<uint64_t>(wp[q + 2]) << (64 - sh);
    const unsigned em = e + m;
    sgn = (win >> em) & 1ull;
    const uint64_t fem = win & ((1ull << em) - 1);
    uint64_t bits = (fem << (52 - m)) + (1023ull << 52);
    if (e == 11) {  // min(offset + 1023, 2046): only an 11-bit offset can exceed it
        if ((fem >> m) >= 1024) bits = (2046ull << 52) | ((fem << (52 - m)) & ((1ull << 52) - 1));
    }
    return __longlong_as_double(static_cast<long long>(bits)) - 1.0;
}

__device__ __forceinline__ double signed_coef(double c, uint64_t sgn) {
    return __longlong_as_double(__double_as_longlong(c) ^ static_cast<long long>(sgn << 63));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ring of kNStage stage buffers fed by cp.async.bulk
struct Ring {
    uint8_t* buf;
    uint64_t* bars;
    __device__ __forceinline__ uint32_t* stage_words(int slot) const {
        return reinterpret_cast<uint32_t*>(buf + slot * (kStageBytes + kSlack));
    }
};

__device__ __forceinline__ void issue_stage(const Params& p, const Ring& r, uint32_t s, int slot,
                                            uint64_t policy) {
    const Stage st = p.stages[s];
    mbar_expect_tx(&r.bars[slot], st.bytes);
    bulk_g2s(r.buf + slot * (kStageBytes + kSlack), p.arena + st.byte_off, st.bytes, &r.bars[slot], policy);
}

// ------------------------------------------------------------ phase A ----
__device__ __forceinline__ void a_item(const Params& p, const AItem& it, const uint32_t* sw,
                                       unsigned lane) {
    const LeafA L = p.leafa[it.leaf];
    const unsigned nf = it.nf;
    double xv[kAChunk / 32];
#pragma unroll
    for (int u = 0; u < kAChunk / 32; ++u) {
        const unsigned f = lane + 32u * u;
        xv[u] = f < nf ? __ldg(p.x + it.xidx + f) : 0.0;
    }
    const uint32_t* wp = sw + it.word_off;
    for (unsigned c = 0; c < it.nseg; ++c) {
        const uint32_t j = it.xcol + c;
        const uint16_t wm = __ldg(p.colx_wm + j);
        const unsigned w = wm & 0xffu, m = wm >> 8;
        const unsigned bit = lane * w, q = bit >> 5, sh = bit & 31u;
        double acc = 0.0;
#pragma unroll
        for (int u = 0; u < kAChunk / 32; ++u) {
            if (lane + 32u * u < nf) {
                uint64_t sg;
                const double a = decode_a(wp, q + u * w, sh, w, L.e, m, sg);
                acc = fma(a, signed_coef(xv[u], sg), acc);
            }
        }
        acc = warp_sum(acc);
        if (lane == 0) {
            if (L.nchunks == 1)
                p.c[j] = p.alpha * __ldg(p.coef + j) * acc;
            else
                p.partial[L.pbase + static_cast<uint32_t>(it.chunk) * L.k + it.icol0 + c] = acc;
        }
        wp += (nf * w + 31) >> 5;
    }
    if (L.nchunks > 1) {
        __threadfence();
        __syncwarp();
        unsigned last = 0;
        if (lane == 0) last = atomicAdd(p.counter + it.leaf, 1u) == L.nitems - 1;
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {  // every chunk is in: sum in fixed chunk order (deterministic)
            __threadfence();
            for (unsigned i = lane; i < L.k; i += 32) {
                double s = 0.0;
                for (unsigned ch = 0; ch < L.nchunks; ++ch) s += __ldcg(p.partial + L.pbase + ch * L.k + i);
                p.c[L.colbase + i] = p.alpha * __ldg(p.coef + L.colbase + i) * s;
            }
            if (lane == 0) p.counter[it.leaf] = 0u;  // re-armed for the next product
        }
    }
}

__global__ void __launch_bounds__(kNW * 32) k_phase_a(Params p) {
    extern __shared__ __align__(128) uint8_t smem[];
    Ring r{smem, reinterpret_cast<uint64_t*>(smem + kNStage * (kStageBytes + kSlack))};
    const unsigned tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t s0 = p.stripe_a[blockIdx.x], s1 = p.stripe_a[blockIdx.x + 1];
    uint64_t policy = 0;
    if (tid == 0) {
        policy = evict_first_policy();
        for (int b = 0; b < kNStage; ++b) mbar_init(&r.bars[b], 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (tid == 0)
        for (int b = 0; b < kNStage && s0 + b < s1; ++b) issue_stage(p, r, s0 + b, b, policy);
    for (uint32_t s = s0; s < s1; ++s) {
        const uint32_t it = s - s0;
        const int slot = static_cast<int>(it % kNStage);
        mbar_wait(&r.bars[slot], (it / kNStage) & 1u);
        const Stage st = p.stages[s];
        const uint32_t* sw = r.stage_words(slot);
        for (uint32_t i = warp; i < st.nitems; i += kNW) a_item(p, p.aitems[st.item0 + i], sw, lane);
        __syncthreads();
        if (tid == 0 && s + kNStage < s1) issue_stage(p, r, s + kNStage, slot, policy);
    }
}

// ------------------------------------------------------------ phase B ----
__global__ void __launch_bounds__(kNW * 32) k_phase_b(Params p) {
    extern __shared__ __align__(128) uint8_t smem[];
    Ring r{smem, reinterpret_cast<uint64_t*>(smem + kNStage * (kStageBytes + kSlack))};
    double* red = reinterpret_cast<double*>(smem + kNStage * (kStageBytes + kSlack) + 64);
    const unsigned tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t blk = blockIdx.x;
    const uint32_t s0 = p.stripe_b[blk], s1 = p.stripe_b[blk + 1];
    const unsigned nrows = p.row_count[blk];
    const bool v0 = lane < nrows, v1 = lane + 32 < nrows;
    uint64_t policy = 0;
    if (tid == 0) {
        policy = evict_first_policy();
        for (int b = 0; b < kNStage; ++b) mbar_init(&r.bars[b], 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (tid == 0)
        for (int b = 0; b < kNStage && s0 + b < s1; ++b) issue_stage(p, r, s0 + b, b, policy);
    double acc0 = 0.0, acc1 = 0.0;
    for (uint32_t s = s0; s < s1; ++s) {
        const uint32_t it = s - s0;
        const int slot = static_cast<int>(it % kNStage);
        mbar_wait(&r.bars[slot], (it / kNStage) & 1u);
        const Stage st = p.stages[s];
        const uint32_t* sw = r.stage_words(slot);
        for (uint32_t i = warp; i < st.nitems; i += kNW) {
            const BItem item = p.bitems[st.item0 + i];
            const uint32_t* wp = sw + item.word_off;
            const unsigned e = item.e;
            if (item.kind == 0) {
                const DenseInfo di = p.dense[item.b];
                const unsigned w = di.w, m = di.m;
                const unsigned bit = lane * w, q = bit >> 5, sh = bit & 31u;
                const unsigned segw = (nrows * w + 31) >> 5;
                double i0 = 0.0, i1 = 0.0;
                for (unsigned c = 0; c < item.nseg; ++c) {
                    const double xc = __ldg(p.x + item.a + c);
                    uint64_t sg;
                    if (v0) i0 = fma(decode_a(wp, q, sh, w, e, m, sg), signed_coef(xc, sg), i0);
                    if (v1) i1 = fma(decode_a(wp, q + w, sh, w, e, m, sg), signed_coef(xc, sg), i1);
                    wp += segw;
                }
                const double mul = p.alpha * di.scale;
                acc0 = fma(mul, i0, acc0);
                acc1 = fma(mul, i1, acc1);
            } else {
                for (unsigned c = 0; c < item.nseg; ++c) {
                    const uint32_t j = item.a + c;
                    const uint16_t wm = __ldg(p.colw_wm + j);
                    const unsigned w = wm & 0xffu, m = wm >> 8;
                    const double cj = p.c[j];
                    const unsigned bit = lane * w, q = bit >> 5, sh = bit & 31u;
                    uint64_t sg;
                    if (v0) acc0 = fma(decode_a(wp, q, sh, w, e, m, sg), signed_coef(cj, sg), acc0);
                    if (v1) acc1 = fma(decode_a(wp, q + w, sh, w, e, m, sg), signed_coef(cj, sg), acc1);
                    wp += (nrows * w + 31) >> 5;
                }
            }
        }
        __syncthreads();
        if (tid == 0 && s + kNStage < s1) issue_stage(p, r, s + kNStage, slot, policy);
    }
    red[warp * 64 + lane] = acc0;
    red[warp * 64 + lane + 32] = acc1;
    __syncthreads();
    if (tid < nrows) {
        double sum = 0.0;
#pragma unroll
        for (int wv = 0; wv < kNW; ++wv) sum += red[wv * 64 + tid];
        double* yp = p.y + p.row_first[blk] + tid;
        *yp = p.beta == 0.0 ? sum : fma(p.beta, *yp, sum);
    }
}

__global__ void k_scale(double* y, uint64_t n, double beta) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += gridDim.x * (uint64_t)blockDim.x)
        y[i] = beta == 0.0 ? 0.0 : beta * y[i];
}

constexpr size_t kSmemBytes = kNStage * (kStageBytes + kSlack) + 64 + kNW * 64 * sizeof(double);

// ------------------------------------------------------- host: layout ----
// copy nbits starting at bit `bit` of the LSB-first stream src[0, len) into
// whole 32-bit words at dst (fields keep their bits; missing bytes read 0)
void copy_bits(const uint8_t* src, uint64_t len, uint64_t bit, uint64_t nbits, uint32_t* dst) {
    const uint64_t nw = (nbits + 31) / 32;
    for (uint64_t t = 0; t < nw; ++t) {
        const uint64_t b = bit + 32 * t;
        const uint64_t byte = b >> 3;
        uint64_t v = 0;
        if (byte + 8 <= len) {
            std::memcpy(&v, src + byte, 8);
        } else {
            for (uint64_t i = 0; i < 8 && byte + i < len; ++i) v |= static_cast<uint64_t>(src[byte + i]) << (8 * i);
        }
        uint32_t word = static_cast<uint32_t>(v >> (b & 7));
        const uint64_t rem = nbits - 32 * t;
        if (rem < 32) word &= (1u << rem) - 1u;
        dst[t] = word;
    }
}

struct SegRef {  // where a run of a buffer's fields landed in the arena (export)
    uint64_t word;  // arena word index
    uint32_t f0, nf;
};

}  // namespace
}  // namespace hcmx_gpu

using namespace hcmx_gpu;

struct hcmx_hmat {
    uint64_t n_rows = 0, n_cols = 0, rb = 0, re = 0;
    DevBuf arena, stages, bitems, aitems, stripe_a, stripe_b, row_first, row_count, leafa, dense, colw, colx,
        coef, c, partial, counter, xbuf, ybuf;
    uint32_t nstripe_a = 0, nblocks = 0, nlr = 0;
    hcmx_memory_report report{};
    std::vector<std::vector<SegRef>> segs;  // per buffer (export); empty if too big
    std::vector<hcmx_descriptor> desc;
    std::vector<int64_t> count;
    cudaStream_t stream = nullptr;
    int last_launches = 0;
    bool timing = false;
    std::vector<cudaEvent_t> ev_pool;
    struct Rec {
        cudaEvent_t a0, a1, b1;
    };
    std::vector<Rec> pending;
    double ms_a = 0, ms_b = 0;
    uint64_t calls = 0;
};

namespace {

cudaEvent_t take_event(hcmx_hmat* h) {
    if (!h->ev_pool.empty()) {
        cudaEvent_t e = h->ev_pool.back();
        h->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    check_cuda(cudaEventCreate(&e), "cudaEventCreate");
    return e;
}

void drain_timing(hcmx_hmat* h) {
    for (auto& r : h->pending) {
        check_cuda(cudaEventSynchronize(r.b1), "cudaEventSynchronize");
        float a = 0, b = 0;
        check_cuda(cudaEventElapsedTime(&a, r.a0, r.a1), "elapsed");
        check_cuda(cudaEventElapsedTime(&b, r.a1, r.b1), "elapsed");
        h->ms_a += a;
        h->ms_b += b;
        h->ev_pool.push_back(r.a0);
        h->ev_pool.push_back(r.a1);
        h->ev_pool.push_back(r.b1);
    }
    h->pending.clear();
}

struct Builder {
    const hcmx_hmat_desc& d;
    hcmx_hmat* h;
    std::vector<uint8_t> blob_host;
    const uint8_t* blob = nullptr;

    std::vector<uint32_t> arena;  // words
    std::vector<Stage> stages;
    std::vector<BItem> bitems;
    std::vector<AItem> aitems;

    Builder(const hcmx_hmat_desc& dd, hcmx_hmat* hh) : d(dd), h(hh) {}

    unsigned width(uint64_t b) const { return d.desc[b].bit_width; }

    // append words of fields [f0, f0+nf) of buffer b; returns words appended
    uint64_t put_fields(uint64_t b, uint64_t f0, uint64_t nf, bool keep_map) {
        const unsigned w = width(b);
        const uint64_t nw = (nf * w + 31) / 32;
        const uint64_t at = arena.size();
        arena.resize(at + nw);
        copy_bits(blob + d.poff[b], static_cast<uint64_t>(d.plen[b]), f0 * w, nf * w, arena.data() + at);
        if (keep_map) h->segs[b].push_back({at, static_cast<uint32_t>(f0), static_cast<uint32_t>(nf)});
        return nw;
    }

    // greedy stage packing over a list of items whose sizes are known; returns
    // for each item its stage-relative word offset
    struct Packer {
        Builder& B;
        uint64_t stage_start_word = 0;
        uint32_t cur_items = 0, item0 = 0;
        bool open = false;
        explicit Packer(Builder& b) : B(b) {}
        void begin(uint32_t first_item) {
            // stages start 16-byte aligned
            while (B.arena.size() % 4) B.arena.push_back(0u);
            stage_start_word = B.arena.size();
            item0 = first_item;
            cur_items = 0;
            open = true;
        }
        // called before writing an item of `words` words; may close/open a stage
        uint32_t place(uint64_t words, uint32_t item_index) {
            if (!open) begin(item_index);
            const uint64_t used = B.arena.size() - stage_start_word;
            if (cur_items > 0 && (used + words) * 4 > static_cast<uint64_t>(kStageBytes)) {
                close();
                begin(item_index);
            }
            if (words * 4 > static_cast<uint64_t>(kStageBytes)) throw invalid_argument("hmat: item exceeds a stage");
            ++cur_items;
            return static_cast<uint32_t>(B.arena.size() - stage_start_word);
        }
        void close() {
            if (!open) return;
            while (B.arena.size() % 4) B.arena.push_back(0u);
            Stage s{};
            s.byte_off = stage_start_word * 4;
            s.bytes = static_cast<uint32_t>((B.arena.size() - stage_start_word) * 4);
            s.item0 = item0;
            s.nitems = cur_items;
            if (s.nitems) B.stages.push_back(s);
            open = false;
        }
    };
};

void validate(const hcmx_hmat_desc& d) {
    if (!d.n_rows || !d.n_cols) throw invalid_argument("hmat: empty matrix");
    if (d.n_rows >= (1ull << 31) || d.n_cols >= (1ull << 31)) throw invalid_argument("hmat: dimension too large");
    for (uint64_t l = 0; l < d.nleaves; ++l) {
        if (d.row0[l] < 0 || d.row1[l] > (int64_t)d.n_rows || d.row0[l] >= d.row1[l] || d.col0[l] < 0 ||
            d.col1[l] > (int64_t)d.n_cols || d.col0[l] >= d.col1[l])
            throw invalid_argument("hmat: leaf range outside the matrix");
        const int64_t rows = d.row1[l] - d.row0[l], cols = d.col1[l] - d.col0[l];
        if (d.kind[l] == 0) {
            if (d.buf0[l] < 0 || d.buf0[l] >= (int64_t)d.nbuffers) throw invalid_argument("hmat: buffer index");
            if (d.count[d.buf0[l]] != rows * cols) throw invalid_argument("hmat: dense leaf size mismatch");
        } else if (d.kind[l] == 1) {
            const int64_t k = d.rank[l];
            if (k < 0 || d.buf0[l] < 0 || d.buf0[l] + 2 * k > (int64_t)d.nbuffers || d.sig0[l] < 0 ||
                d.sig0[l] + k > (int64_t)d.nsigma)
                throw invalid_argument("hmat: lowrank leaf indices");
            for (int64_t i = 0; i < k; ++i) {
                if (d.count[d.buf0[l] + i] != rows || d.count[d.buf0[l] + k + i] != cols)
                    throw invalid_argument("hmat: lowrank factor size mismatch");
            }
        } else {
            throw invalid_argument("hmat: unsupported leaf kind (only CodecDense and APLRLowrank)");
        }
    }
    for (uint64_t b = 0; b < d.nbuffers; ++b) {
        const hcmx_descriptor& x = d.desc[b];
        if (x.scheme > 3 || x.exp_bits < 2 || x.exp_bits > 11 || x.mant_bits < 2 || x.mant_bits > 52 ||
            x.bit_width != bit_width(x.scheme, x.exp_bits, x.mant_bits))
            throw invalid_argument("hmat: invalid buffer descriptor");
        if (d.poff[b] < 0 || d.plen[b] < 0 || (uint64_t)(d.poff[b] + d.plen[b]) > d.blob_bytes)
            throw corrupt_buffer("hmat: payload outside the blob");
        if ((uint64_t)d.plen[b] < payload_bytes(d.count[b], x.bit_width))
            throw corrupt_buffer("bitstream: payload ends inside a value");
    }
}

void build(const hcmx_hmat_desc& d, hcmx_hmat* h) {
    validate(d);
    Builder B(d, h);
    if (d.blob_on_device) {
        B.blob_host.resize(d.blob_bytes);
        check_cuda(cudaMemcpy(B.blob_host.data(), d.blob, d.blob_bytes, cudaMemcpyDeviceToHost), "blob d2h");
        B.blob = B.blob_host.data();
    } else {
        B.blob = d.blob;
    }
    h->n_rows = d.n_rows;
    h->n_cols = d.n_cols;
    h->rb = d.row_begin;
    h->re = d.row_end;
    if (h->rb == 0 && h->re == 0) h->re = d.n_rows;
    if (h->rb >= h->re || h->re > d.n_rows) throw invalid_argument("hmat: bad row partition");
    h->desc.assign(d.desc, d.desc + d.nbuffers);
    h->count.assign(d.count, d.count + d.nbuffers);

    // leaves that write rows of this partition
    std::vector<uint64_t> leaves;
    for (uint64_t l = 0; l < d.nleaves; ++l)
        if ((uint64_t)d.row0[l] < h->re && (uint64_t)d.row1[l] > h->rb) leaves.push_back(l);

    // row blocks: every leaf boundary, then <= 64 rows each
    std::vector<uint64_t> cuts = {h->rb, h->re};
    for (uint64_t l : leaves) {
        cuts.push_back(std::clamp<uint64_t>(d.row0[l], h->rb, h->re));
        cuts.push_back(std::clamp<uint64_t>(d.row1[l], h->rb, h->re));
    }
    std::sort(cuts.begin(), cuts.end());
    cuts.erase(std::unique(cuts.begin(), cuts.end()), cuts.end());
    std::vector<uint32_t> rfirst, rcount;
    for (size_t i = 0; i + 1 < cuts.size(); ++i)
        for (uint64_t r = cuts[i]; r < cuts[i + 1]; r += kRowBlock) {
            rfirst.push_back(static_cast<uint32_t>(r));
            rcount.push_back(static_cast<uint32_t>(std::min<uint64_t>(kRowBlock, cuts[i + 1] - r)));
        }
    const uint32_t nblocks = static_cast<uint32_t>(rfirst.size());
    std::vector<std::vector<uint32_t>> block_leaves(nblocks);
    for (uint64_t l : leaves) {
        const uint64_t a = std::max<uint64_t>(d.row0[l], h->rb), b = std::min<uint64_t>(d.row1[l], h->re);
        auto it = std::lower_bound(rfirst.begin(), rfirst.end(), static_cast<uint32_t>(a));
        for (; it != rfirst.end() && *it < b; ++it) block_leaves[it - rfirst.begin()].push_back(static_cast<uint32_t>(l));
    }

    // per-leaf tables
    uint64_t total_fields = 0;
    for (uint64_t b = 0; b < d.nbuffers; ++b) total_fields += d.count[b];
    const bool keep_map = total_fields <= (1ull << 28);
    if (keep_map) h->segs.assign(d.nbuffers, {});

    std::vector<int64_t> lr_id(d.nleaves, -1), dense_id(d.nleaves, -1);
    std::vector<LeafA> leafa;
    std::vector<DenseInfo> dense;
    std::vector<uint16_t> colw, colx;
    std::vector<double> coef;
    uint64_t npartial = 0;
    hcmx_memory_report& rep = h->report;
    rep = hcmx_memory_report{};
    for (uint64_t l : leaves) {
        const int64_t rows = d.row1[l] - d.row0[l], cols = d.col1[l] - d.col0[l];
        if (d.kind[l] == 0) {
            const hcmx_descriptor& x = d.desc[d.buf0[l]];
            dense_id[l] = static_cast<int64_t>(dense.size());
            DenseInfo di{};
            di.scale = x.scale;
            di.w = x.bit_width;
            di.m = x.mant_bits;
            di.e = x.exp_bits;
            dense.push_back(di);
            rep.dense_leaves++;
            rep.dense_compressed += 20 + d.plen[d.buf0[l]];
            rep.uncompressed_equivalent += 8ull * rows * cols;
            rep.algorithmic_bytes += 20 + payload_bytes(rows * cols, x.bit_width);
        } else {
            const uint32_t k = static_cast<uint32_t>(d.rank[l]);
            lr_id[l] = static_cast<int64_t>(leafa.size());
            LeafA L{};
            L.colbase = static_cast<uint32_t>(colw.size());
            L.k = k;
            L.nchunks = static_cast<uint32_t>((cols + kAChunk - 1) / kAChunk);
            L.nitems = L.nchunks * ((k + kAGroup - 1) / kAGroup);
            L.pbase = static_cast<uint32_t>(npartial);
            L.e = k ? d.desc[d.buf0[l] + k].exp_bits : 2;
            if (L.nchunks > 1) npartial += static_cast<uint64_t>(L.nchunks) * k;
            leafa.push_back(L);
            uint64_t bytes = 8 + 8ull * k;  // APLRLowrank::byte_size (mixedprec.cpp:210-217)
            for (uint32_t i = 0; i < k; ++i) {
                const hcmx_descriptor& xw = d.desc[d.buf0[l] + i];
                const hcmx_descriptor& xx = d.desc[d.buf0[l] + k + i];
                colw.push_back(static_cast<uint16_t>(xw.bit_width | (xw.mant_bits << 8)));
                colx.push_back(static_cast<uint16_t>(xx.bit_width | (xx.mant_bits << 8)));
                coef.push_back(d.sigma[d.sig0[l] + i] * xx.scale * xw.scale);
                bytes += 40 + d.plen[d.buf0[l] + i] + d.plen[d.buf0[l] + k + i];
                rep.algorithmic_bytes += 40 + payload_bytes(rows, xw.bit_width) + payload_bytes(cols, xx.bit_width);
            }
            rep.algorithmic_bytes += 8ull * k;
            rep.lowrank_leaves++;
            rep.lowrank_compressed += bytes;
            rep.uncompressed_equivalent += 8ull * (rows + cols) * k;
        }
    }
    rep.algorithmic_bytes += 8ull * d.n_cols + 8ull * (h->re - h->rb);
    h->nlr = static_cast<uint32_t>(leafa.size());

    // ---- phase A items / stages / stripes
    std::vector<uint32_t> stripe_a = {0};
    {
        Builder::Packer P(B);
        uint32_t stages_in_stripe = 0;
        for (uint64_t l : leaves) {
            if (d.kind[l] != 1) continue;
            const LeafA& L = leafa[lr_id[l]];
            const int64_t cols = d.col1[l] - d.col0[l];
            for (uint32_t ch = 0; ch < L.nchunks; ++ch) {
                const uint64_t f0 = static_cast<uint64_t>(ch) * kAChunk;
                const uint64_t nf = std::min<uint64_t>(kAChunk, cols - f0);
                for (uint32_t g = 0; g < L.k; g += kAGroup) {
                    const uint32_t ng = std::min<uint32_t>(kAGroup, L.k - g);
                    uint64_t words = 0;
                    for (uint32_t i = g; i < g + ng; ++i) words += (nf * B.width(d.buf0[l] + L.k + i) + 31) / 32;
                    const size_t before = B.stages.size();
                    AItem it{};
                    it.word_off = P.place(words, static_cast<uint32_t>(B.aitems.size()));
                    if (B.stages.size() != before && ++stages_in_stripe >= kAStagesPerStripe) {
                        stripe_a.push_back(static_cast<uint32_t>(B.stages.size()));
                        stages_in_stripe = 0;
                    }
                    it.nseg = static_cast<uint16_t>(ng);
                    it.nf = static_cast<uint16_t>(nf);
                    it.xcol = L.colbase + g;
                    it.xidx = static_cast<uint32_t>(d.col0[l] + f0);
                    it.leaf = static_cast<uint32_t>(lr_id[l]);
                    it.chunk = static_cast<uint16_t>(ch);
                    it.icol0 = static_cast<uint16_t>(g);
                    for (uint32_t i = g; i < g + ng; ++i) B.put_fields(d.buf0[l] + L.k + i, f0, nf, keep_map);
                    B.aitems.push_back(it);
                }
            }
        }
        P.close();
        if (stripe_a.back() != B.stages.size()) stripe_a.push_back(static_cast<uint32_t>(B.stages.size()));
    }
    rep.stages_a = B.stages.size();

    // ---- phase B items / stages, one stripe per row block
    std::vector<uint32_t> stripe_b = {static_cast<uint32_t>(B.stages.size())};
    for (uint32_t blk = 0; blk < nblocks; ++blk) {
        Builder::Packer P(B);
        const uint64_t r0 = rfirst[blk], nr = rcount[blk];
        for (uint32_t l : block_leaves[blk]) {
            const int64_t rows = d.row1[l] - d.row0[l], cols = d.col1[l] - d.col0[l];
            const uint64_t roff = r0 - d.row0[l];
            if (d.kind[l] == 0) {
                const uint64_t b = d.buf0[l];
                const unsigned w = B.width(b);
                for (int64_t c0 = 0; c0 < cols; c0 += kBDenseGroup) {
                    const uint32_t nc = static_cast<uint32_t>(std::min<int64_t>(kBDenseGroup, cols - c0));
                    BItem it{};
                    it.word_off = P.place(nc * ((nr * w + 31) / 32), static_cast<uint32_t>(B.bitems.size()));
                    it.nseg = static_cast<uint16_t>(nc);
                    it.kind = 0;
                    it.e = d.desc[b].exp_bits;
                    it.a = static_cast<uint32_t>(d.col0[l] + c0);
                    it.b = static_cast<uint32_t>(dense_id[l]);
                    for (uint32_t c = 0; c < nc; ++c) B.put_fields(b, (c0 + c) * rows + roff, nr, keep_map);
                    B.bitems.push_back(it);
                }
            } else {
                const LeafA& L = leafa[lr_id[l]];
                for (uint32_t g = 0; g < L.k; g += kBLRGroup) {
                    const uint32_t ng = std::min<uint32_t>(kBLRGroup, L.k - g);
                    uint64_t words = 0;
                    for (uint32_t i = g; i < g + ng; ++i) words += (nr * B.width(d.buf0[l] + i) + 31) / 32;
                    BItem it{};
                    it.word_off = P.place(words, static_cast<uint32_t>(B.bitems.size()));
                    it.nseg = static_cast<uint16_t>(ng);
                    it.kind = 1;
                    it.e = L.k ? d.desc[d.buf0[l]].exp_bits : 2;
                    it.a = L.colbase + g;
                    it.b = 0;
                    for (uint32_t i = g; i < g + ng; ++i) B.put_fields(d.buf0[l] + i, roff, nr, keep_map);
                    B.bitems.push_back(it);
                }
            }
        }
        P.close();
        stripe_b.push_back(static_cast<uint32_t>(B.stages.size()));
    }
    rep.stages_b = B.stages.size() - rep.stages_a;
    // B items index their own array: rebase B stage item0 (A and B share `stages`)
    // (A stages reference aitems, B stages reference bitems -- item0 is per array)
    while (B.arena.size() % 4) B.arena.push_back(0u);
    B.arena.resize(B.arena.size() + 8, 0u);  // tail slack

    // ---- upload
    cudaStream_t s = h->stream;
    auto up = [&](DevBuf& dst, const void* src, size_t bytes) {
        dst.alloc(std::max<size_t>(bytes, 16));
        if (bytes) h2d(dst.p, src, bytes, s);
    };
    up(h->arena, B.arena.data(), B.arena.size() * 4);
    up(h->stages, B.stages.data(), B.stages.size() * sizeof(Stage));
    up(h->bitems, B.bitems.data(), B.bitems.size() * sizeof(BItem));
    up(h->aitems, B.aitems.data(), B.aitems.size() * sizeof(AItem));
    up(h->stripe_a, stripe_a.data(), stripe_a.size() * 4);
    up(h->stripe_b, stripe_b.data(), stripe_b.size() * 4);
    up(h->row_first, rfirst.data(), rfirst.size() * 4);
    up(h->row_count, rcount.data(), rcount.size() * 4);
    up(h->leafa, leafa.data(), leafa.size() * sizeof(LeafA));
    up(h->dense, dense.data(), dense.size() * sizeof(DenseInfo));
    up(h->colw, colw.data(), colw.size() * 2);
    up(h->colx, colx.data(), colx.size() * 2);
    up(h->coef, coef.data(), coef.size() * 8);
    h->c.alloc(std::max<size_t>(16, coef.size() * 8));
    h->partial.alloc(std::max<size_t>(16, npartial * 8));
    h->counter.alloc(std::max<size_t>(16, leafa.size() * 4));
    check_cuda(cudaMemsetAsync(h->counter.p, 0, h->counter.bytes, s), "memset");
    stream_sync(s);
    h->nstripe_a = static_cast<uint32_t>(stripe_a.size() - 1);
    h->nblocks = nblocks;
    rep.device_arena_bytes = B.arena.size() * 4;
    rep.device_table_bytes = B.stages.size() * sizeof(Stage) + B.bitems.size() * sizeof(BItem) +
                             B.aitems.size() * sizeof(AItem) + leafa.size() * sizeof(LeafA) +
                             dense.size() * sizeof(DenseInfo) + colw.size() * 12 + coef.size() * 16;
    rep.overhead = rep.device_table_bytes;
}

Params make_params(hcmx_hmat* h, double alpha, const double* x, double beta, double* y) {
    Params p{};
    p.arena = h->arena.as<uint8_t>();
    p.stages = h->stages.as<Stage>();
    p.bitems = h->bitems.as<BItem>();
    p.aitems = h->aitems.as<AItem>();
    p.stripe_a = h->stripe_a.as<uint32_t>();
    p.stripe_b = h->stripe_b.as<uint32_t>();
    p.row_first = h->row_first.as<uint32_t>();
    p.row_count = h->row_count.as<uint32_t>();
    p.leafa = h->leafa.as<LeafA>();
    p.dense = h->dense.as<DenseInfo>();
    p.colw_wm = h->colw.as<uint16_t>();
    p.colx_wm = h->colx.as<uint16_t>();
    p.coef = h->coef.as<double>();
    p.c = h->c.as<double>();
    p.partial = h->partial.as<double>();
    p.counter = h->counter.as<unsigned>();
    p.x = x;
    p.y = y;
    p.alpha = alpha;
    p.beta = beta;
    return p;
}

void run_matvec(hcmx_hmat* h, double alpha, const double* dx, double beta, double* dy, cudaStream_t s) {
    static bool attr_set = false;
    if (!attr_set) {
        check_cuda(cudaFuncSetAttribute(k_phase_a, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes),
                   "smem attr");
        check_cuda(cudaFuncSetAttribute(k_phase_b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes),
                   "smem attr");
        attr_set = true;
    }
    h->last_launches = 0;
    if (alpha == 0.0) {  // y = beta y without touching M
        const uint64_t n = h->re - h->rb;
        k_scale<<<(int)std::min<uint64_t>((n + 255) / 256, 4096), 256, 0, s>>>(dy + h->rb, n, beta);
        check_cuda(cudaGetLastError(), "scale launch");
        h->last_launches = 1;
        return;
    }
    Params p = make_params(h, alpha, dx, beta, dy);
    hcmx_hmat::Rec rec{};
    if (h->timing) {
        rec = {take_event(h), take_event(h), take_event(h)};
        check_cuda(cudaEventRecord(rec.a0, s), "event");
    }
    if (h->nlr && h->nstripe_a) {
        k_phase_a<<<h->nstripe_a, kNW * 32, kSmemBytes, s>>>(p);
        h->last_launches++;
    }
    if (h->timing) check_cuda(cudaEventRecord(rec.a1, s), "event");
    if (h->nblocks) {
        k_phase_b<<<h->nblocks, kNW * 32, kSmemBytes, s>>>(p);
        h->last_launches++;
    }
    check_cuda(cudaGetLastError(), "matvec launch");
    if (h->timing) {
        check_cuda(cudaEventRecord(rec.b1, s), "event");
        h->pending.push_back(rec);
        h->calls++;
        if (h->pending.size() > 1024) drain_timing(h);
    }
}

}  // namespace

extern "C" {

int hcmx_gpu_hmat_create(const hcmx_hmat_desc* desc, hcmx_hmat** out) {
    return guarded([&] {
        require_device();
        auto* h = new hcmx_hmat();
        try {
            check_cuda(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking), "cudaStreamCreate");
            build(*desc, h);
        } catch (...) {
            if (h->stream) cudaStreamDestroy(h->stream);
            delete h;
            throw;
        }
        *out = h;
    });
}

int hcmx_gpu_hmat_destroy(hcmx_hmat* h) {
    return guarded([&] {
        if (!h) return;
        cudaStreamSynchronize(h->stream);
        for (auto& r : h->pending) {
            cudaEventDestroy(r.a0);
            cudaEventDestroy(r.a1);
            cudaEventDestroy(r.b1);
        }
        for (auto e : h->ev_pool) cudaEventDestroy(e);
        cudaStreamDestroy(h->stream);
        delete h;
    });
}

int hcmx_gpu_hmat_memory(const hcmx_hmat* h, hcmx_memory_report* out) {
    return guarded([&] { *out = h->report; });
}

int hcmx_gpu_hmat_matvec_device(hcmx_hmat* h, double alpha, const double* d_x, double beta, double* d_y,
                                void* stream) {
    return guarded([&] { run_matvec(h, alpha, d_x, beta, d_y, (cudaStream_t)stream); });
}

int hcmx_gpu_hmat_matvec(hcmx_hmat* h, double alpha, const double* h_x, double beta, double* h_y,
                         int transpose) {
    return guarded([&] {
        if (transpose) throw invalid_argument("matvec: transpose is not supported");
        if (!h->xbuf.p) h->xbuf.alloc(h->n_cols * 8);
        if (!h->ybuf.p) h->ybuf.alloc(h->n_rows * 8);
        const uint64_t nr = h->re - h->rb;
        h2d(h->xbuf.p, h_x, h->n_cols * 8, h->stream);
        if (beta != 0.0) h2d(h->ybuf.as<double>() + h->rb, h_y + h->rb, nr * 8, h->stream);
        run_matvec(h, alpha, h->xbuf.as<double>(), beta, h->ybuf.as<double>(), h->stream);
        d2h(h_y + h->rb, h->ybuf.as<double>() + h->rb, nr * 8, h->stream);
        stream_sync(h->stream);
    });
}

int hcmx_gpu_hmat_export_buffer(const hcmx_hmat* h, uint64_t b, uint8_t* h_payload, uint64_t capacity,
                                uint64_t* len) {
    return guarded([&] {
        if (h->segs.empty()) throw invalid_argument("export: segment map not kept for this matrix size");
        if (b >= h->segs.size()) throw invalid_argument("export: buffer index");
        const unsigned w = h->desc[b].bit_width;
        const uint64_t n = payload_bytes(h->count[b], w);
        if (n > capacity) throw invalid_argument("export: capacity");
        std::vector<uint8_t> bits(n + 16, 0);
        for (const SegRef& sref : h->segs[b]) {
            const uint64_t nw = (static_cast<uint64_t>(sref.nf) * w + 31) / 32;
            std::vector<uint32_t> words(nw);
            check_cuda(cudaMemcpy(words.data(), h->arena.as<uint32_t>() + sref.word, nw * 4, cudaMemcpyDeviceToHost),
                       "export d2h");
            // OR the fields back at their original bit offset
            const uint64_t base = static_cast<uint64_t>(sref.f0) * w;
            for (uint64_t bit = 0; bit < static_cast<uint64_t>(sref.nf) * w; ++bit) {
                if ((words[bit >> 5] >> (bit & 31)) & 1u) {
                    const uint64_t o = base + bit;
                    bits[o >> 3] |= static_cast<uint8_t>(1u << (o & 7));
                }
            }
        }
        std::memcpy(h_payload, bits.data(), n);
        *len = n;
    });
}

int hcmx_gpu_hmat_last_launches(const hcmx_hmat* h) { return h ? h->last_launches : 0; }

int hcmx_gpu_hmat_timing(hcmx_hmat* h, int enable, double* ms_a, double* ms_b, uint64_t* calls) {
    return guarded([&] {
        drain_timing(h);
        if (ms_a) *ms_a = h->ms_a;
        if (ms_b) *ms_b = h->ms_b;
        if (calls) *calls = h->calls;
        if (enable >= 0) {  // enable < 0: query only
            h->timing = enable != 0;
            h->ms_a = h->ms_b = 0;
            h->calls = 0;
        }
    });
}

}  // extern "C"
