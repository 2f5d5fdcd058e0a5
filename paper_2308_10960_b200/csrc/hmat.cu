// hmat.cu -- device-resident compressed H-matrix and the fused
// decompress + matrix-vector product (hmatrix.hpp:126-128).
//
// Layout (built once on the host by hcmx_gpu_hmat_create):
//   The packed codec fields of every leaf are re-tiled, each field keeping its
//   bits, into one HBM arena of 16-byte aligned stages.  A stage is one bulk
//   copy (TMA engine) into a shared-memory ring slot; its staged coefficients
//   follow it in the slot.  Stages are grouped into stripes that persistent
//   CTAs claim from a global counter (largest estimated cost first).
//
//   phase A (lowrank X^T x): item = up to 32 lanes, one 64-row chunk of one X
//     column per lane, row-interleaved (row j = the lanes' fields back to
//     back, groups of 4 rows padded to whole words).  Each lane sums its own
//     column -- no cross-lane reduction; consecutive chunks of one column
//     (<= 8, a segment) are summed by a fixed in-warp butterfly, wider leaves
//     leave one partial per segment for k_reduce.
//   phase B (row-stationary): one stripe = one block of 128 rows and every
//     item that writes those rows: dense leaves and the W slices of every
//     lowrank leaf covering the block, column-major.  Lane l owns rows
//     32 g + l (4 accumulators per warp); the CTA sums its warps once at the
//     end and writes y once per row -- no atomics.
//
//   One producer warp per CTA fills a 3-slot ring (stage data with L2
//   evict_first, coefficient copies); consumer warps decode from shared
//   memory only.  A field costs two LDS, one funnel shift, a mask, one wide
//   IMAD, one DADD, one LOP3 for the sign and one DFMA (dec_fast).
//
// Numerics: decoded values are bit-identical to codec::decompress_into; the
// multiply by the buffer scale is folded into the coefficients (dense: alpha *
// scale * x_j, lowrank: alpha * sigma_i * scale_X_i * scale_W_i * t_i), so the
// sum differs from the oracle only by FP64 reassociation (||dy||/||y|| ~ 1e-15).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <sys/mman.h>

#include <cstdio>
#include <cstdlib>

#ifndef HCMX_WAIT_HINT
#define HCMX_WAIT_HINT 200
#endif

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "internal.h"
#include <type_traits>

namespace hcmx_gpu {
namespace {

#ifndef HCMX_NWB
#define HCMX_NWB 8
#endif
constexpr int kNWB = HCMX_NWB;            // phase-B consumer warps per CTA
#ifndef HCMX_NWA
#define HCMX_NWA 8
#endif
#ifndef HCMX_NWB_MULTI
#define HCMX_NWB_MULTI 8
#endif
// phase B: a 2-slot ring of 45 KB stages (measured against 3 x 26 KB, 4 x 17 KB and
// 2 x 40 / 43 KB: the per-stage bookkeeping of the consumer warps costs more than
// the shallower ring; config 4's phase B 2.29 -> 2.17 ms)
#ifndef HCMX_NSTAGE
#define HCMX_NSTAGE 2
#endif
#ifndef HCMX_STAGE_BYTES
#define HCMX_STAGE_BYTES 46080
#endif
constexpr int kNWA = HCMX_NWA;            // phase-A consumer warps (more registers per thread)
#ifndef HCMX_COSCHED
#define HCMX_COSCHED 0
#endif
#ifndef HCMX_AMINB
#define HCMX_AMINB 2
#endif
#ifndef HCMX_BMINB
#define HCMX_BMINB 2
#endif
constexpr int kCtasA = HCMX_AMINB, kCtasB = HCMX_BMINB;  // resident CTAs per SM (persistent grids)
// The coefficient copies of a stage (x slices, phase-A results: ~12 small bulk
// copies per phase-A stage, each an ELECT / R2UR round trip of ~130 clocks) are
// issued by a second producer warp; the first one issues the stage's one large
// copy and runs the stage sequence.  (One producer warp was busy 88 % of phase A
// and the consumer warps waited for data 23 % of it.)
#ifndef HCMX_COEF_WARP
#define HCMX_COEF_WARP 1
#endif
constexpr int kNProd = HCMX_COEF_WARP ? 2 : 1;  // producer warps per CTA
constexpr int kThreadsA = (kNWA + kNProd) * 32;
constexpr int kStageBytes = HCMX_STAGE_BYTES;  // packed data per stage
constexpr int kMaxItems = 32;             // items per stage (one per producer lane)
constexpr int kItemBytes = 32;            // descriptor size (A and B)
constexpr int kCoefBytes = 7936;          // staged coefficients + column params per stage
constexpr int kNStage = HCMX_NSTAGE;      // ring depth (phase B)
#ifndef HCMX_NSTAGE_A
#define HCMX_NSTAGE_A 3  // phase A keeps 3 x 26 KB (2 x 43 KB measured slower)
#endif
constexpr int kNStageA = HCMX_NSTAGE_A;   // ring depth of phase A (its CTAs need no reduction buffer)
template <bool PHASE_A>
__host__ __device__ constexpr int nstage() { return PHASE_A ? kNStageA : kNStage; }
constexpr int kSlack = 16;                // decode reads up to 2 words past a segment
constexpr unsigned kWaitHintNs = HCMX_WAIT_HINT;  // mbarrier try_wait suspend hint (ns)
// A stage is one contiguous arena range, copied by ONE bulk copy into the slot:
// [items (32 B each)][phase B: per-warp item ranges, 48 B][packed data]; its
// staged coefficients (x slices, phase-A results) follow it in the same slot,
// at the 16-byte aligned end of the stage, so a stage may trade packed data
// for coefficients (phase A's x slices are ~1/3 of its packed bytes).  The
// builder bakes slot-relative coefficient offsets into the items.
constexpr int kStageMax = kMaxItems * kItemBytes + 64 + kStageBytes;
constexpr int kSlotData = kStageMax + kSlack + kCoefBytes;  // stage + coefficients
constexpr int kOffHdr = kSlotData;    // slot header written by the producer: stripe id, flags,
                                      // item claim counter (phase A), items
constexpr int kSlotBytes = kOffHdr + 16;
// phase A may use its own (smaller) stages: HCMX_STAGE_BYTES_A / HCMX_COEF_BYTES_A
#ifndef HCMX_STAGE_BYTES_A
#define HCMX_STAGE_BYTES_A 26624
#endif
#ifndef HCMX_COEF_BYTES_A
#define HCMX_COEF_BYTES_A 7936
#endif
constexpr int kStageBytesA = HCMX_STAGE_BYTES_A;
constexpr int kStageMaxA = kMaxItems * kItemBytes + 64 + kStageBytesA;
constexpr int kSlotDataA = kStageMaxA + kSlack + HCMX_COEF_BYTES_A;
constexpr int kOffHdrA = kSlotDataA;
constexpr int kSlotBytesA = kOffHdrA + 16;
static_assert(kOffHdrA % 16 == 0 && kSlotBytesA % 16 == 0, "phase-A slot alignment");
template <bool PHASE_A>
__host__ __device__ constexpr int slot_bytes() { return PHASE_A ? kSlotBytesA : kSlotBytes; }
template <bool PHASE_A>
__host__ __device__ constexpr int off_hdr() { return PHASE_A ? kOffHdrA : kOffHdr; }
constexpr int kR = 128;               // rows per phase-B CTA
constexpr int kG = kR / 32;           // row groups (accumulators) per lane
#ifndef HCMX_A_SIGMA
#define HCMX_A_SIGMA 1
#endif
#ifndef HCMX_A_STATIC
#define HCMX_A_STATIC 1
#endif
#ifndef HCMX_ACHUNK
#define HCMX_ACHUNK 64  // 32 measured: phase A 0.122 -> 0.136 ms (the per-item work doubles)
#endif
constexpr int kAChunk = HCMX_ACHUNK;  // rows of a leaf's X columns per phase-A chunk
constexpr int kARows = 4;             // rows per word-padded group of a phase-A item
constexpr int kALanes = 32;           // rank columns per phase-A item
#ifndef HCMX_AGROUP
#define HCMX_AGROUP 8
#endif
constexpr int kAGroupMax = HCMX_AGROUP;  // chunks of one rank column summed in-warp
#ifndef HCMX_AGROUP_MULTI
#define HCMX_AGROUP_MULTI 2
#endif
constexpr uint32_t kAGroupMaxMulti = HCMX_AGROUP_MULTI;  // the same for multi-RHS arenas
#ifndef HCMX_AUNROLL
#define HCMX_AUNROLL 4
#endif
#ifndef HCMX_AITEM
#define HCMX_AITEM 8192
#endif
constexpr int kAUnroll = HCMX_AUNROLL;   // row groups per iteration of the phase-A fast body
constexpr uint64_t kAItemBytes = HCMX_AITEM;  // packed data per phase-A item
constexpr uint32_t kAItemXBytes = 12288;  // staged x slices per phase-A item
#ifndef HCMX_BLR_UNROLL
#define HCMX_BLR_UNROLL 2
#endif
constexpr int kBLRUnroll = HCMX_BLR_UNROLL;  // columns per iteration of the phase-B lowrank body (R = 1) on 4 row groups; twice as many on 2
#ifndef HCMX_BGROUP
#define HCMX_BGROUP 32
#endif
#ifndef HCMX_BITEM
#define HCMX_BITEM 8192
#endif
constexpr int kBLRGroup = HCMX_BGROUP;  // max columns per B item
#ifndef HCMX_ASTRIPE
#define HCMX_ASTRIPE 32
#endif
constexpr uint64_t kAStripeBytes = HCMX_ASTRIPE * 26624ull;  // target packed bytes per phase-A stripe (one CTA's claim)
constexpr uint64_t kItemTarget = 1536;          // packed bytes per item (columns grouped up to this)
constexpr uint64_t kItemMaxBytes = HCMX_BITEM;  // items merge columns up to this many packed bytes
constexpr size_t kRingBytes = static_cast<size_t>(kNStage) * kSlotBytes;
constexpr size_t kRingBytesA = static_cast<size_t>(kNStageA) * kSlotBytesA;
constexpr size_t kRedBytes = ((kNWB > HCMX_NWB_MULTI ? kNWB : HCMX_NWB_MULTI) / 2) * kR * sizeof(double);  // phase-B cross-warp reduction
constexpr int kMailSlots = 8;  // stage indices published by the first producer warp for the second
constexpr size_t kMailBytes = (kMailSlots + 2) * sizeof(uint32_t) + 8;  // + published / read counters, padding
constexpr size_t kSmemBytes = kRingBytes + kRedBytes + 2 * kNStage * sizeof(uint64_t) + kMailBytes;  // + full, empty barriers
constexpr size_t kSmemBytesA = kRingBytesA + 2 * kNStageA * sizeof(uint64_t) + kMailBytes;
static_assert(kNStage + 2 <= kMailSlots && kNStageA + 2 <= kMailSlots, "mailbox depth");
constexpr int kCopies = 2 * kMaxItems;  // coefficient copies per stage (two per producer lane)
constexpr int kRangeBytes = 64;         // phase-B stage head: 16 warp item ranges (begin | end << 16)
// copy entry (u64): [0,32) source element index, [32,48) dst / 16 in the slot,
// [48,60) bytes / 16, [60,62) source table (0 x, 1 wcol records), bit 63 valid
static_assert(kOffHdr % 16 == 0 && kSlotBytes % 16 == 0, "slot alignment");
constexpr uint32_t kHdrLast = 1u, kHdrEnd = 2u, kHdrEmpty = 4u;  // slot header flags

struct Stage {
    uint64_t byte_off;   // packed data in the arena
    uint32_t bytes;
    uint32_t item0;      // first descriptor (A or B array); grouped by warp
    uint32_t nitems;
    uint32_t coef_bytes; // bytes of staged coefficients / params (exact sum of the copies)
    uint64_t pad;
};
static_assert(sizeof(Stage) == 32, "Stage layout");

// Column layout parameters of the fast decoder (dec_fast), precomputed on the
// host: the field's e + m bits once it is left-aligned (bits [32 - w, 31)) and
// the multiplier 2^(21 + e) that moves them to bits [52 - m, 52 + e)
struct ColPar {
    uint32_t mask;       // ((1 << (w - 1)) - 1) << (32 - w)
    uint32_t mul;        // 1 << (21 + e)
    uint32_t packed;     // w | m << 8 | e << 16 | mode << 24 (mode 0 fast, 2 generic, 3-5 raw)
    uint32_t w;
};

// One rank column of a lowrank leaf as phase B needs it (32 bytes, two
// LDS.128): the phase-A result c_i = alpha coef_i (X_i^T x), written each
// product, and the W column's decoder constants, precomputed at build time.
// A leaf's records are contiguous, so one bulk copy stages a whole leaf.
struct WCol {
    double c;
    uint32_t mask, mul, packed, w, pad0, pad1;
};
static_assert(sizeof(WCol) == 32, "WCol layout");

// Products with R right-hand sides at once (decode once, R FMAs per value):
// rank-column records carry R phase-A results, {double c[R]; mask, mul,
// packed, w}, 16-byte aligned; R = 1 is the WCol layout above.
template <int R>
__host__ __device__ constexpr int rec_bytes() { return R == 1 ? 32 : (8 * R + 16 + 15) / 16 * 16; }
constexpr uint32_t kMaxPieces = 4;  // pieces a phase-B row block may be split into
constexpr int kMultiR = 4;    // right-hand sides per product of a multi-RHS arena
constexpr int kMultiR2 = 8;   // ... of the wide multi-RHS arena (nrhs_block = 8)
constexpr int kNWBMulti = HCMX_NWB_MULTI;  // phase-B consumer warps for R > 1 (R x 4 accumulators per lane)
inline uint32_t rec_bytes_rt(int R) { return R == 1 ? 32u : static_cast<uint32_t>((8 * R + 16 + 15) / 16 * 16); }
template <int R>
__host__ __device__ constexpr int nwb() { return R == 1 ? HCMX_NWB : (R == 4 ? kNWBMulti : 6); }  // R = 8: 4 R accumulators per lane

struct BItem {
    uint32_t word_off;   // packed data, from the warp-stage start
    uint8_t nseg;        // columns in this item
    uint8_t kind;        // 0 dense, 1 lowrank
    uint8_t ra;          // first row of the item inside the row block
    uint8_t nr;          // rows (fields per column segment)
    uint32_t coef_off;   // staged coefficient of the first column (x or phase-A result), coef-area bytes
    uint32_t src;        // dense: x index of first column; lowrank: global W column id
    uint32_t dpacked;    // dense: w | m << 8 | e << 16 | mode << 24
    uint8_t mode;        // decode mode shared by every column of the item
    uint8_t fcase;       // decode body (bcase_of): 1-3 fast (whole row groups), 0 generic
    uint16_t pad;
    double scale;        // dense: buffer scale
};
static_assert(sizeof(BItem) == kItemBytes, "BItem layout");

// A phase-A item: up to 32 rank columns ("lanes") with the same number of rows
// nf -- the X columns of one or more leaf chunks.  Lane l owns column l and
// sums X_l^T x over its rows by itself (no cross-lane reduction).  The data is
// row-interleaved: row j holds the fields of lanes 0..nl-1 back to back (row
// width rowbits = sum of the lane widths), and every group of kARows rows is
// padded to whole words, so a lane's field sits at the same (word, shift) in
// every group.  Ahead of the data: one 32-bit record per lane (aligned to 16
// bytes): w | e << 7 | m << 11 | fmt << 17 | x offset in the slot (doubles) << 19,
// fmt 0 codec field, 1-3 uncompressed FP64 / FP32 / FP16.
struct AItem {
    uint32_t word_off;   // lane records, then the data groups (words from the stage start)
    uint16_t nf;         // rows (fields per lane)
    uint8_t nl;          // lanes, 1..32
    uint8_t body;        // 1: fast body (every lane w <= 32, e <= 10, codec fields), 0: generic
    uint32_t dest0;      // lane l writes element dest0 + l (wcol record or partial)
    uint16_t rowbits;    // bits per row (sum of the lane widths)
    uint16_t gwords;     // words per group of kARows rows
    uint8_t final_;      // 1: c = alpha coef (X^T x) into wcol; 0: partial sum (k_reduce)
    uint8_t cshift;      // 2^cshift column slots; lane l = g * 2^cshift + slot holds chunk g of
                         // its slot's rank column (the chunks are summed in-warp)
    uint8_t pad[14];
};
static_assert(sizeof(AItem) == kItemBytes, "AItem layout");

struct LeafA {  // host-side only
    uint32_t colbase;   // global column id of rank column 0
    uint32_t k;
    uint32_t pbase;     // partials base (nchunks > 1)
    uint32_t nchunks;
};

struct Params {
    const uint8_t* arena;
    const Stage* stages;
    const uint4* stripe_a;      // [nstripe_a] {stage begin, end, -, -}, most expensive first
    const uint4* stripe_b;      // [nstripe_b] {stage begin, end, row block, piece}, most expensive first;
                                // piece 0: the whole block, writes y; piece q > 0: part q - 1 of a
                                // block split across CTAs, writes ypart (k_combine adds the parts)
    const uint64_t* copies;     // [nstages * kCopies] staged coefficient copies (see CopyEntry)
    unsigned* work;             // [2] stripe counters of the persistent kernels (A, B), zeroed per product
    uint32_t nstripe_a, nblocks;  // nblocks: phase-B stripes (row blocks or their pieces)
    double* ypart;              // [pieces][local rows][R] partial row sums of split blocks
    const double* coef;         // sigma_i * scale_X_i * scale_W_i
    uint8_t* wrec;              // per rank column: record {c[R], mask, mul, packed, w} (rec_bytes<R>):
                                // c = alpha * coef * (X^T x) per right-hand side (phase A) + W decoder constants
    double* partial;
    const double* x2;           // complex arenas: the swapped right-hand sides (-Im x, Re x) per pair
    const double* x;            // R = 1: padded internal copy (16-byte aligned, readable + 16 B);
                                // R > 1: n x R, row-major (the R right-hand sides interleaved)
    double* y;                  // R > 1: n x R, row-major
    uint32_t row_begin, row_end;
    double alpha, beta;
    uint64_t bias;              // 1023 << 52, the decoders' exponent bias: a runtime value keeps it in
                                // a register pair (a literal is rematerialised into uniform registers
                                // inside every decode loop)
    int debug;                  // profiling knob (HCMX_DEBUG): 1 = consumers skip the decode
};

// ------------------------------------------------------- instrumentation --
// HCMX_PROF builds only: per-phase cycle counters (consumer wait / busy,
// producer wait on free slots / total), read back by the host when HCMX_PROF is
// set in the environment.  [phase][0 wait_full, 1 busy, 2 prod_wait_empty,
// 3 prod_total, 4 consumer warps, 5 stripe-end cycles, 6 CTA ns, 7 CTAs]
#ifdef HCMX_PROF
__device__ unsigned long long g_prof[2][8];
__device__ unsigned long long g_ts[2][4];  // min start, max end, sum end, sum start (ns, globaltimer)
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define PROF_ADD(ph, i, v) atomicAdd(&g_prof[ph][i], static_cast<unsigned long long>(v))
#else
#define PROF_ADD(ph, i, v) ((void)0)
#endif
#ifdef HCMX_PROF
__device__ __forceinline__ long long clk() { return clock64(); }
#else
__device__ __forceinline__ long long clk() { return 0; }  // no clock reads in product builds
#endif

// the HCMX_DEBUG profiling knob reaches the kernels in HCMX_PROF builds only
#ifdef HCMX_PROF
#define dbg(p) ((p).debug)
#else
#define dbg(p) 0
#endif

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
__device__ __forceinline__ void bulk_g2s_plain(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, unsigned parity) {
    uint32_t ok;
#if HCMX_WAIT_HINT > 0
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(kWaitHintNs)  // short suspend instead of a hot spin
        : "memory");
#else
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
#endif
    return ok != 0;
}

// A wait that never completes (a byte count the copies do not deliver) traps
// after ~seconds instead of hanging the device: the launch fails with an error.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    uint32_t n = 0;
    while (!mbar_try_wait(bar, parity)) {
        if (++n == (1u << 26)) __trap();
    }
}

// Programmatic dependent launch: k_reduce and k_phase_b are launched while the
// kernel before them still runs (their CTAs take SMs as phase-A CTAs retire)
// and wait for its completion only where they first read what it wrote.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}



// ------------------------------------------------------------- decode ----
// A field's layout is [mant m][offset e][sign] (codec.cpp:118-137); every
// decoder returns +-((1.mant * 2^offset) - 1) -- exactly the codec's value /
// scale (codec.cpp:161-169).
//
// Fast decoder (w == 1 + e + m <= 32, e <= 10, codec fields): with `top` the
// stream bit one past the field's sign bit, hi is word top >> 5 and lo the word
// below it; the right funnel shift by top (mod 32) brings stream bits [top - 32,
// top) into one register: the field left-aligned, sign in bit 31 (top a
// multiple of 32: the shift is 0 and lo is the result).  Neither the word index
// nor the shift needs top - 1 or a negation.  The offset and mantissa bits
// times 2^(21 + e) land at bits [52 - m, 52 + e) of the double, so one wide
// IMAD with the bias 1023 << 52 rebuilds 1.mant * 2^offset (offset + 1023 <=
// 2046: no clamp for e <= 10); one DADD takes the 1 off and the sign is xored
// into the high word.  About 8 instructions per value with the FMA.
__device__ __forceinline__ double dec_pair(uint32_t lo, uint32_t hi, unsigned s, uint32_t mask, uint32_t mul,
                                          uint64_t bias) {
    const uint32_t t = __funnelshift_r(lo, hi, s);
    const uint64_t bits = static_cast<uint64_t>(t & mask) * mul + bias;
    const double v = __longlong_as_double(static_cast<long long>(bits)) - 1.0;
    return __hiloint2double(__double2hiint(v) ^ static_cast<int>(t & 0x80000000u), __double2loint(v));
}

// top >> 5 kept as a shift (an opaque one: the compiler otherwise rewrites the
// scaled vector index into shift + mask + add, one instruction more per column)
__device__ __forceinline__ unsigned word_of(unsigned top) {
    unsigned r;
    asm("shr.u32 %0, %1, 5;" : "=r"(r) : "r"(top));
    return r;
}

// Interleaved word streams: NG streams (row groups of a column segment, or the
// 4 rows of a phase-A group) whose word j sits at NG j + g, so the two words a
// field needs in every stream come with two NG-word vector loads (LDS.128 for
// NG = 4, LDS.64 for NG = 2) from one address.  q: the stream words' vector
// base (16- / 8-byte aligned), o: the word below the fields' sign words (may
// be -1: the bits it brings are masked off; the word above may lie one vector
// past the stream, inside the slot: it is shifted out).
template <int NG>
__device__ __forceinline__ void il_load(const uint32_t* q, int o, uint32_t (&lo)[NG], uint32_t (&hi)[NG]) {
    static_assert(NG == 2 || NG == 4, "interleave");
    if constexpr (NG == 4) {
        const uint4* v = reinterpret_cast<const uint4*>(q) + o;
        const uint4 a = v[0], b = v[1];
        lo[0] = a.x, lo[1] = a.y, lo[2] = a.z, lo[3] = a.w;
        hi[0] = b.x, hi[1] = b.y, hi[2] = b.z, hi[3] = b.w;
    } else {
        const uint2* v = reinterpret_cast<const uint2*>(q) + o;
        const uint2 a = v[0], b = v[1];
        lo[0] = a.x, lo[1] = a.y;
        hi[0] = b.x, hi[1] = b.y;
    }
}

// Generic decoder: the field at bit sh of sp[0], sp[st], sp[2 st] (64-bit window, the
// min(offset + 1023, 2046) clamp), for e = 11, w > 32 and padded layouts;
// modes 3, 4, 5: uncompressed FP64 / FP32 / FP16 storage (StorageMode fp64 and
// the MP-D-S-H groups, mixedprec.hpp:20-43), the value itself (scale 1).
__device__ __forceinline__ double dec_generic(const uint32_t* sp, uint32_t packed, unsigned sh, unsigned st = 1) {
    const unsigned fmt = packed >> 24;
    const unsigned w = packed & 0xffu, m = (packed >> 8) & 0xffu, e = (packed >> 16) & 0xffu;
    uint64_t win = ((static_cast<uint64_t>(sp[st]) << 32) | sp[0]) >> sh;
    if (w > 32 && sh + w > 64) win |= static_cast<uint64_t>(sp[2 * st]) << (64 - sh);
    if (fmt >= 3) {  // uncompressed words (uniform per item, so the branch is too)
        if (fmt == 3)  // FP64
            return __longlong_as_double(static_cast<long long>(win));
        if (fmt == 4)  // FP32
            return static_cast<double>(__int_as_float(static_cast<int>(static_cast<uint32_t>(win))));
        // binary16 (the half.hpp:47-72 widening is exact)
        const uint32_t t = static_cast<uint32_t>(win) & 0xffffu;
        return static_cast<double>(__half2float(__ushort_as_half(static_cast<unsigned short>(t))));
    }
    const unsigned em = e + m;
    const uint64_t sgn = (win >> em) & 1ull;
    const uint64_t fem = win & ((1ull << em) - 1);
    uint64_t bits = (fem << (52 - m)) + (1023ull << 52);
    if ((fem >> m) >= 1024) bits = (2046ull << 52) | ((fem << (52 - m)) & ((1ull << 52) - 1));
    const double d = __longlong_as_double(static_cast<long long>(bits)) - 1.0;
    return __longlong_as_double(__double_as_longlong(d) ^ static_cast<long long>(sgn << 63));
}

// 2^(21 + e), read from a table: a multiplier the compiler cannot see is a
// power of two stays one wide IMAD (fused with the exponent bias) instead of a
// 64-bit shift pair plus a 64-bit add on the integer pipe
struct Pow2Table {
    uint32_t v[32];
};
constexpr Pow2Table make_pow2e() {
    Pow2Table t{};
    for (int e = 0; e < 32; ++e) t.v[e] = e <= 10 ? (1u << (21 + e)) : 0u;
    return t;
}
__constant__ Pow2Table c_pow2e = make_pow2e();

// fast-decoder constants from a layout word (w <= 32)
__device__ __forceinline__ uint32_t fast_mask(unsigned w) { return 0x7fffffffu & ~((0xffffffffu >> (w - 1)) >> 1); }




// ------------------------------------------------------- warp pipeline ----


// One warp fills the ring: the stage's packed data, its item descriptors and
// per-warp ranges, and -- per item, one item per lane -- the coefficient slice
// (x or the phase-A results) plus the column parameters, all as cp.async.bulk
// copies completing on the slot's full barrier.  Consumers never wait on global
// memory.  The metadata of stage s+1 is fetched while waiting for a free slot.
template <int R>
__device__ __forceinline__ void issue_copy(const Params& p, uint64_t c, uint8_t* cdst, uint64_t* bar) {
    if (!(c >> 63)) return;
    const uint32_t idx = static_cast<uint32_t>(c);
    const unsigned dst = static_cast<unsigned>((c >> 32) & 0xffffu) * 16u;
    const unsigned bytes = static_cast<unsigned>((c >> 48) & 0xfffu) * 16u;
    const void* src;
    switch (static_cast<unsigned>((c >> 60) & 3u)) {
        case 0: src = p.x + static_cast<size_t>(idx) * R; break;
        case 2: src = p.x2 + static_cast<size_t>(idx) * R; break;  // complex: swapped x
        default: src = p.wrec + static_cast<size_t>(idx) * rec_bytes<R>(); break;
    }
    bulk_g2s_plain(cdst + dst, src, bytes, bar);
}

// Stage sequence of a persistent CTA: stripes are claimed one at a time from a
// global counter (any CTA may take any stripe; every stripe's result is the
// same whoever computes it, so the product stays deterministic).  A stripe is
// claimed only when the previous one is exhausted (claiming ahead would hold
// stripes back from idle CTAs at the tail).
struct StageSeq {
    uint32_t stripe = 0, s = 0, e = 0;  // stage s of stripe [.., e)
    bool done = false;
};

template <bool PHASE_A>
__device__ __forceinline__ void seq_next(const Params& p, StageSeq& q, unsigned lane) {
    if (q.done) return;
    if (q.s + 1 < q.e) {
        ++q.s;
        return;
    }
    const uint32_t nstripes = PHASE_A ? p.nstripe_a : p.nblocks;
    for (;;) {
        uint32_t id = 0;
        if (lane == 0) id = atomicAdd(p.work + (PHASE_A ? 0 : 1), 1u);
        id = __shfl_sync(0xffffffffu, id, 0);
        if (id >= nstripes) {
            q.done = true;
            return;
        }
        const uint4 r = (PHASE_A ? p.stripe_a : p.stripe_b)[id];
        if (r.x < r.y || !PHASE_A) {  // phase B visits empty row blocks too (y = beta y)
            q.stripe = id;
            q.s = r.x;
            q.e = r.y;
            return;
        }
    }
}

struct StageMeta {  // what the producer needs for one stage, loaded ahead
    Stage st;
    uint64_t c0, c1;
    uint32_t stripe;
    uint32_t flags;  // kHdrLast / kHdrEnd
    uint32_t sidx;   // stage index (kMailEnd / kMailSkip for header-only stages): what the second producer warp is told
    bool empty;      // a row block without stages: header only
};
constexpr uint32_t kMailEnd = 0xffffffffu, kMailSkip = 0xfffffffeu;

// mailbox between the two producer warps (shared memory): seq[it % kMailSlots]
// = stage index of the CTA's it-th stage, pub = stages published, rd = stages read
struct Mail {
    uint32_t seq[kMailSlots];
    uint32_t pub, rd;
};
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}
__device__ __forceinline__ void spin_until_ge(const uint32_t* p, uint32_t v) {
    uint32_t n = 0;
    while (static_cast<int32_t>(ld_acquire(p) - v) < 0) {
        __nanosleep(20);
        if (++n == (1u << 26)) __trap();
    }
}

template <bool PHASE_A>
__device__ __forceinline__ StageMeta seq_meta(const Params& p, const StageSeq& q, unsigned lane) {
    StageMeta m{};
    if (q.done) {
        m.flags = kHdrEnd;
        m.sidx = kMailEnd;
        return m;
    }
    m.stripe = q.stripe;
    if (q.s >= q.e) {  // empty phase-B row block
        m.empty = true;
        m.flags = kHdrLast | kHdrEmpty;
        m.sidx = kMailSkip;
        return m;
    }
    m.st = p.stages[q.s];
    m.sidx = q.s;
    if (kNProd == 1) {
        m.c0 = __ldg(p.copies + static_cast<size_t>(q.s) * kCopies + lane);
        m.c1 = __ldg(p.copies + static_cast<size_t>(q.s) * kCopies + 32 + lane);
    }
    m.flags = q.s + 1 == q.e ? kHdrLast : 0u;
    return m;
}

// One warp fills the ring: per stage the packed data, the item descriptors,
// the per-warp ranges and the coefficient / column-parameter copies (a fixed
// stride list of <= 64 copy entries per stage, two per lane), all completing
// on the slot's full barrier, plus a small header (stripe id, last-stage and
// end flags) written before the copies.  The metadata of every stage is loaded
// two stages ahead, so no global load sits on the producer's critical path.
template <bool PHASE_A, int R>
__device__ __forceinline__ void producer(const Params& p, uint8_t* ring, uint64_t* full, uint64_t* empty,
                                         Mail* mail, unsigned lane) {
    const uint64_t policy = evict_first_policy();
    StageSeq q;
    q.s = q.e = 0;
    uint32_t npub = 0;  // stages published to the second producer warp
    auto publish = [&](const StageMeta& m) {
        if (kNProd == 1) return;
        if (lane == 0) {
            if (npub >= kMailSlots) spin_until_ge(&mail->rd, npub - kMailSlots + 1);  // the entry overwritten was read
            mail->seq[npub % kMailSlots] = m.sidx;
            st_release(&mail->pub, npub + 1);
        }
        ++npub;
    };
    seq_next<PHASE_A>(p, q, lane);
    StageMeta mx = seq_meta<PHASE_A>(p, q, lane);
    publish(mx);
    seq_next<PHASE_A>(p, q, lane);
    StageMeta my = seq_meta<PHASE_A>(p, q, lane);
    publish(my);
    StageMeta mz;
    const long long t_start = clk();
#ifdef HCMX_PROF
    const unsigned long long g0 = gtime();
#endif
    long long t_wait = 0;
    bool waited = false;           // phase B: griddepcontrol.wait done
    constexpr int NS = nstage<PHASE_A>();
    unsigned slot = 0, phase = 0;  // it % NS, parity of the slot's previous use
    uint32_t it = 0;
    // one stage: issue `cur`, load the metadata of the stage two ahead into
    // `ahead` (three rotating registers sets: no register copy waits on a load)
    auto step = [&](const StageMeta& cur, StageMeta& ahead) -> bool {
        seq_next<PHASE_A>(p, q, lane);
        ahead = seq_meta<PHASE_A>(p, q, lane);
        publish(ahead);
        const long long t0 = clk();
        if (it >= NS) mbar_wait(&empty[slot], phase);
        t_wait += clk() - t0;
        uint8_t* base = ring + static_cast<size_t>(slot) * slot_bytes<PHASE_A>();
        if (lane == 0) {
            uint32_t* hdr = reinterpret_cast<uint32_t*>(base + off_hdr<PHASE_A>());
            hdr[0] = cur.stripe;
            hdr[1] = cur.flags;
            hdr[2] = 0u;  // item claim counter
            hdr[3] = (cur.flags & kHdrEnd || cur.empty) ? 0u : cur.st.nitems;
        }
        __syncwarp();
        if (cur.flags & kHdrEnd || cur.empty) {  // header only
            if (lane == 0) mbar_arrive(&full[slot]);
        } else {
            if (!PHASE_A && !waited && kNProd == 1) {
                // the first stage that copies phase-A column coefficients (table
                // 1) waits for phase A and k_reduce to complete; dense stages
                // before it run while they drain
                const bool needs_a = ((cur.c0 >> 63) && ((cur.c0 >> 60) & 3u) == 1u) ||
                                     ((cur.c1 >> 63) && ((cur.c1 >> 60) & 3u) == 1u);
                if (__any_sync(0xffffffffu, needs_a)) {
                    pdl_wait();
                    waited = true;
                }
            }
            const bool no_coef = dbg(p) >= 2;  // profiling knob
            if (lane == 0) {
                mbar_expect_tx(&full[slot], cur.st.bytes + (no_coef ? 0u : cur.st.coef_bytes));
                bulk_g2s(base, p.arena + cur.st.byte_off, cur.st.bytes, &full[slot], policy);
            }
            __syncwarp();
            if (!no_coef && kNProd == 1) {
                issue_copy<R>(p, cur.c0, base, &full[slot]);
                issue_copy<R>(p, cur.c1, base, &full[slot]);
            }
        }
        if (cur.flags & kHdrEnd) {
            if (!PHASE_A && blockIdx.x == 0 && lane == 0) {
                if (!waited) pdl_wait();
                p.work[0] = 0u;  // phase A's stripe counter, for the next product
            }
            if (lane == 0) {
                PROF_ADD(PHASE_A ? 0 : 1, 2, t_wait);
                PROF_ADD(PHASE_A ? 0 : 1, 3, clk() - t_start);
                PROF_ADD(PHASE_A ? 0 : 1, 7, 1);
#ifdef HCMX_PROF
                const unsigned long long g1 = gtime();
                atomicMin(&g_ts[PHASE_A ? 0 : 1][0], g0);
                atomicMax(&g_ts[PHASE_A ? 0 : 1][1], g1);
                atomicAdd(&g_ts[PHASE_A ? 0 : 1][2], g1 >> 8);
                atomicAdd(&g_ts[PHASE_A ? 0 : 1][3], g0 >> 8);
#endif
            }
            return true;
        }
        ++it;
        if (++slot == NS) {
            slot = 0;
            if (it > NS) phase ^= 1u;
        }
        return false;
    };
    for (;;) {
        if (step(mx, mz)) return;
        if (step(my, mx)) return;
        if (step(mz, my)) return;
    }
}

// The second producer warp: the coefficient copies of every stage, in the
// stage order the first producer warp publishes (two stages ahead of its own
// copies, so the copy entries are loaded before the slot is free).  Both warps
// wait for the slot's empty barrier; the first one posts the expected bytes of
// all the stage's copies (a copy that lands before that only drives the
// barrier's transaction count negative until the expect arrives -- the phase
// cannot complete before the producer's arrival).
template <bool PHASE_A, int R>
__device__ __forceinline__ void coef_producer(const Params& p, uint8_t* ring, uint64_t* full, uint64_t* empty,
                                              Mail* mail, unsigned lane) {
    constexpr int NS = nstage<PHASE_A>();
    const bool no_coef = dbg(p) >= 2;
    unsigned slot = 0, phase = 0;
    uint32_t it = 0;
    bool waited = false;  // phase B: griddepcontrol.wait done by this warp
    auto fetch = [&](uint32_t i, uint32_t& sidx, uint64_t& c0, uint64_t& c1) {
        spin_until_ge(&mail->pub, i + 1);
        sidx = mail->seq[i % kMailSlots];
        __syncwarp();
        if (lane == 0) st_release(&mail->rd, i + 1);
        c0 = c1 = 0;
        if (sidx < kMailSkip) {
            c0 = __ldg(p.copies + static_cast<size_t>(sidx) * kCopies + lane);
            c1 = __ldg(p.copies + static_cast<size_t>(sidx) * kCopies + 32 + lane);
        }
    };
    uint32_t sx, sy;
    uint64_t x0, x1, y0, y1;
    fetch(0, sx, x0, x1);
    auto step = [&](uint32_t cur, uint64_t c0, uint64_t c1, uint32_t& nsidx, uint64_t& n0, uint64_t& n1) -> bool {
        if (cur == kMailEnd) return true;
        fetch(it + 1, nsidx, n0, n1);  // the next stage's entries are in flight during this one's copies
        if (cur != kMailSkip && !no_coef) {
            if (it >= NS) mbar_wait(&empty[slot], phase);
            if (!PHASE_A && !waited) {
                // the first stage that copies phase-A column coefficients (table
                // 1) waits for phase A and k_reduce to complete; dense stages
                // before it run while they drain
                const bool needs_a = ((c0 >> 63) && ((c0 >> 60) & 3u) == 1u) || ((c1 >> 63) && ((c1 >> 60) & 3u) == 1u);
                if (__any_sync(0xffffffffu, needs_a)) {
                    pdl_wait();
                    waited = true;
                }
            }
            uint8_t* base = ring + static_cast<size_t>(slot) * slot_bytes<PHASE_A>();
            issue_copy<R>(p, c0, base, &full[slot]);
            issue_copy<R>(p, c1, base, &full[slot]);
        }
        ++it;
        if (++slot == NS) {
            slot = 0;
            if (it > NS) phase ^= 1u;
        }
        return false;
    };
    for (;;) {
        if (step(sx, x0, x1, sy, y0, y1)) return;
        if (step(sy, y0, y1, sx, x0, x1)) return;
    }
}

// consumer warps of a persistent CTA: body(slot_base, first, end) for the
// warp's items of every stage; at the last stage of a stripe, stripe_end(id)
// DYN (phase A: every item writes its own results, so any assignment gives
// the same bits): the stage's items are dealt round-robin to the warps, the
// deal rotated by one warp per stage (HCMX_A_STATIC = 1, the default; with 0
// the warps claim the items one at a time with a shared-memory atomic, which
// measured 3-5 % slower: a claim and its shuffle per item and per stage visit).
// Otherwise each warp takes its precomputed contiguous range (phase B: a
// warp's row sums must see the same items in the same order on every run:
// deterministic y).
// one item claim: a plain shared-memory atomic from one lane (atomicAdd from a
// lane-0 branch compiles to the warp-aggregated sequence, ~12 instructions)
__device__ __forceinline__ unsigned claim(uint32_t* counter) {
    unsigned v;
    asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(v) : "r"(smem_u32(counter)) : "memory");
    return v;
}

template <int NW, bool DYN, class Body, class End>
__device__ __forceinline__ void consume(uint8_t* ring, uint64_t* full, uint64_t* empty, unsigned warp,
                                        unsigned lane, int debug, Body&& body, End&& stripe_end) {
    long long t_wait = 0, t_busy = 0, t_end = 0;
    constexpr int NS = nstage<DYN>();  // DYN consumers are phase A's
    unsigned slot = 0, phase = 0;  // ring position of stage it: it % NS, (it / NS) & 1
    unsigned rot = 0;              // stage count modulo NW (static item deal)
    for (;;) {
        const long long t0 = clk();
        mbar_wait(&full[slot], phase);
        const long long t1 = clk();
        t_wait += t1 - t0;
        const uint8_t* base = ring + static_cast<size_t>(slot) * slot_bytes<DYN>();
        uint32_t* hdr = reinterpret_cast<uint32_t*>(ring + static_cast<size_t>(slot) * slot_bytes<DYN>() + off_hdr<DYN>());
        const uint32_t stripe = hdr[0], flags = hdr[1];
        if (flags & kHdrEnd) {
            if (lane == 0) {
                PROF_ADD(DYN ? 0 : 1, 0, t_wait);
                PROF_ADD(DYN ? 0 : 1, 1, t_busy);
                PROF_ADD(DYN ? 0 : 1, 4, 1);
                PROF_ADD(DYN ? 0 : 1, 5, t_end);
            }
            return;
        }
        if (debug) {
#if HCMX_A_STATIC
        } else if (DYN) {
            // items of a stage dealt round-robin to the warps, the deal rotated by
            // one warp per stage (items are sorted largest first); every item
            // writes its own results, so any assignment gives the same bits
            const unsigned n = hdr[3];
            for (unsigned i = (warp + NW - rot) % NW; i < n; i += NW) body(base, i);
            rot = rot + 1 == NW ? 0u : rot + 1;
        } else if (false) {
#else
        } else if (DYN) {
#endif
            // the next claim is issued before the current item is decoded, so the
            // shared atomic's latency hides behind it
            const unsigned n = hdr[3];
            unsigned nl = 0;
            if (lane == 0) nl = claim(hdr + 2);
            unsigned i = __shfl_sync(0xffffffffu, nl, 0);
            while (i < n) {
                if (lane == 0) nl = claim(hdr + 2);
                body(base, i);
                i = __shfl_sync(0xffffffffu, nl, 0);
            }
        } else if (!(flags & kHdrEmpty)) {
            // phase-B stage: [per-warp item ranges, 16 x u32 (begin | end << 16)][items][data]
            const uint32_t r = reinterpret_cast<const uint32_t*>(base)[warp];
            for (unsigned i = r & 0xffffu, e = r >> 16; i < e; ++i) body(base, i);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        const long long t2 = clk();
        t_busy += t2 - t1;
        if (flags & kHdrLast) {
            stripe_end(stripe);
            t_end += clk() - t2;
        }
        if (++slot == NS) {
            slot = 0;
            phase ^= 1u;
        }
    }
}

template <int NW, int NS>
__device__ __forceinline__ void ring_init(uint64_t* full, uint64_t* empty, Mail* mail) {
    if (threadIdx.x == 0) {
        mail->pub = mail->rd = 0u;
        for (int b = 0; b < NS; ++b) {
            mbar_init(&full[b], 1);
            mbar_init(&empty[b], NW);
        }
        fence_barrier_init();
    }
    __syncthreads();
}

// ------------------------------------------------------------ phase A ----
// Item data: groups of kARows rows; each row is the lanes' fields back to back
// (rowbits), padded to whole words, and the kARows rows of a group are
// word-interleaved (row r's word j at 4 j + r; gwords = 4 * row words), so a
// lane's field sits at the same (word, shift) in every row: the two words of
// its four fields in a group come with two LDS.128.
// Fast body: every lane's field is a codec field with w <= 32 and e <= 10
// (dec_pair), the item has whole row groups and every lane's x slice is
// 16-byte aligned.  xs: this lane's x rows, R values per row.  R = 1 keeps one
// FMA chain per row of the group, R > 1 one chain per right-hand side.
template <int R, int NGC = 0>  // NGC > 0: exactly NGC row groups (fully unrolled, no trip count)
__device__ __forceinline__ void a_fast(const uint32_t* data, unsigned P, unsigned w, unsigned e, const double* xs,
                                       unsigned ngroups_rt, unsigned gwords, uint64_t bias, double (&res)[R]) {
    const unsigned ngroups = NGC > 0 ? static_cast<unsigned>(NGC) : ngroups_rt;
    const uint32_t mask = fast_mask(w);
    const uint32_t mul = c_pow2e.v[e & 31u];
    const unsigned top = P + w;                          // one past the field's sign bit (in a row)
    const int o = static_cast<int>(top >> 5) - 1;        // the word below the one holding bit `top`
    const unsigned s = top;                              // the funnel shift takes it modulo 32
    const uint32_t* q = data;
    constexpr int NA = R == 1 ? kARows : R;
    double acc[NA];
#pragma unroll
    for (int i = 0; i < NA; ++i) acc[i] = 0.0;
#pragma unroll (NGC > 0 ? NGC : kAUnroll)
    for (unsigned g = 0; g < ngroups; ++g) {
        uint32_t lo[kARows], hi[kARows];
        il_load<kARows>(q, o, lo, hi);
        if constexpr (R >= 8) {  // the x values row by row (R doubles per row)
#pragma unroll
            for (int r = 0; r < kARows; ++r) {
                const double d = dec_pair(lo[r], hi[r], s, mask, mul, bias);
                const double2* xr = reinterpret_cast<const double2*>(xs) + (kARows * g + r) * (R / 2);
#pragma unroll
                for (int i = 0; i < R / 2; ++i) {
                    const double2 t = xr[i];
                    acc[2 * i] = fma(d, t.x, acc[2 * i]);
                    acc[2 * i + 1] = fma(d, t.y, acc[2 * i + 1]);
                }
            }
        } else {
            double xv[kARows * R];
#pragma unroll
            for (int i = 0; i < kARows * R / 2; ++i) {
                const double2 t = reinterpret_cast<const double2*>(xs)[2 * R * g + i];
                xv[2 * i] = t.x;
                xv[2 * i + 1] = t.y;
            }
#pragma unroll
            for (int r = 0; r < kARows; ++r) {
                const double d = dec_pair(lo[r], hi[r], s, mask, mul, bias);
                if (R == 1) {
                    acc[r] = fma(d, xv[r], acc[r]);
                } else {
#pragma unroll
                    for (int c = 0; c < R; ++c) acc[c % NA] = fma(d, xv[r * R + c], acc[c % NA]);
                }
            }
        }
        q += gwords;
    }
    if (R == 1) res[0] = (acc[0] + acc[1]) + (acc[2 % NA] + acc[3 % NA]);
    else {
#pragma unroll
        for (int c = 0; c < R; ++c) res[c] = acc[c % NA];
    }
}

// Generic body: any layout (e = 11, w > 32, uncompressed words), any row count,
// any x alignment -- the mode-2 decoder per field (row words 4 apart).
template <int R>
__device__ __forceinline__ void a_generic(const uint32_t* data, unsigned P, uint32_t rec, const double* xs,
                                          unsigned nf, unsigned gwords, double (&res)[R]) {
    const unsigned w = rec & 127u, e = (rec >> 7) & 15u, m = (rec >> 11) & 63u, fmt = (rec >> 17) & 3u;
    const uint32_t packed = w | (m << 8) | (e << 16) | ((fmt ? fmt + 2u : 2u) << 24);  // 1-3: raw f64 / f32 / f16
#pragma unroll
    for (int c = 0; c < R; ++c) res[c] = 0.0;
    const uint32_t* row0 = data + 4 * (P >> 5);
    for (unsigned j = 0; j < nf; ++j) {
        const double d = dec_generic(row0 + (j / kARows) * gwords + (j % kARows), packed, P & 31u, kARows);
#pragma unroll
        for (int c = 0; c < R; ++c) res[c] = fma(d, xs[j * R + c], res[c]);
    }
}

template <int R>
__device__ __forceinline__ double* rec_c(const Params& p, uint32_t col) {
    return reinterpret_cast<double*>(p.wrec + static_cast<size_t>(col) * rec_bytes<R>());
}

// the chunks of a slot's rank column (lanes slot, slot + nslot, ...): fixed
// butterfly (lane `slot` gets the same order on every run); idle lanes add 0;
// then the slot lanes write c = alpha coef (X^T x) or the partial sum
template <int R>
__device__ __forceinline__ void a_finish(const Params& p, double (&r)[R], bool act, unsigned lane, unsigned nslot,
                                         unsigned dest, unsigned final_, double cf) {
#pragma unroll
    for (int c = 0; c < R; ++c) {
        if (!act) r[c] = 0.0;
        for (unsigned o = nslot; o < 32u; o <<= 1) r[c] += __shfl_xor_sync(0xffffffffu, r[c], o);
    }
    if (!act || lane >= nslot) return;
    if (final_) {
        double* out = rec_c<R>(p, dest);
#pragma unroll
        for (int c = 0; c < R; ++c) out[c] = p.alpha * cf * r[c];
    } else {
#pragma unroll
        for (int c = 0; c < R; ++c) p.partial[static_cast<size_t>(dest) * R + c] = r[c];
    }
}

// Lane records.  Fast items (AItem::body = 1: every lane a codec field with
// w <= 32, e <= 10, an even x offset): [0,5) w - 1, [5,9) e, [9,19) the lane's bit
// offset inside a row (the exclusive prefix sum of the widths, baked by the
// builder: no 5-round shuffle scan per item), [19,31) x offset / 2 (doubles in
// the slot), bit 31 valid.  Generic items: [0,7) w, [7,11) e, [11,17) m,
// [17,19) format, [19,32) x offset; w = 0 idle.
constexpr uint32_t kARecValid = 0x80000000u;

template <int R>
__device__ __forceinline__ void a_item(const Params& p, const AItem* ip, const uint8_t* slot, unsigned lane) {
    // the descriptor with two loads issued together (word_off | nf, nl, body | dest0 | rowbits, gwords || final_, cshift)
    const uint4 d0 = *reinterpret_cast<const uint4*>(ip);
    const uint32_t d1 = reinterpret_cast<const uint32_t*>(ip)[4];
    const unsigned it_nf = d0.y & 0xffffu, nl = (d0.y >> 16) & 0xffu, it_body = d0.y >> 24;
    const unsigned it_gwords = d0.w >> 16, it_final = d1 & 0xffu, it_cshift = (d1 >> 8) & 0xffu;
    const uint32_t* recs = reinterpret_cast<const uint32_t*>(slot) + d0.x;
    const uint32_t r0 = recs[lane < nl ? lane : 0u];
    const unsigned nslot = 1u << it_cshift;
    const unsigned dest = d0.z + lane;      // written by the slot lanes (g == 0) only
    const uint32_t* data = recs + ((nl + 3u) & ~3u);
    double r[R];
    bool act;
    if (it_body) {
        act = lane < nl && (r0 & kARecValid) != 0u;
        double cf = 0.0;
        if (act && lane < nslot && it_final) cf = __ldg(p.coef + dest);  // in flight during the decode
        const uint32_t rec = act ? r0 : recs[0];  // idle lanes shadow lane 0 (results dropped)
        const unsigned w = (rec & 31u) + 1u, e = (rec >> 5) & 15u, P = (rec >> 9) & 1023u;
        const double* xs = reinterpret_cast<const double*>(slot) + 2u * ((rec >> 19) & 4095u);
        // whole 64-row chunks (most items): the 16 row groups fully unrolled
        if (R == 1 && it_nf == kAChunk) a_fast<R, kAChunk / kARows>(data, P, w, e, xs, 0, it_gwords, p.bias, r);
        else a_fast<R>(data, P, w, e, xs, it_nf / kARows, it_gwords, p.bias, r);
        a_finish<R>(p, r, act, lane, nslot, dest, it_final, cf);
    } else {
        act = lane < nl && (r0 & 127u) != 0u;
        double cf = 0.0;
        if (act && lane < nslot && it_final) cf = __ldg(p.coef + dest);
        const uint32_t rec = act ? r0 : recs[0];
        // this lane's bit offset inside a row: exclusive prefix sum of the widths
        const unsigned w = rec & 127u;
        unsigned P = act ? w : 0u;
#pragma unroll
        for (unsigned o = 1; o < 32; o <<= 1) {
            const unsigned v = __shfl_up_sync(0xffffffffu, P, o);
            if (lane >= o) P += v;
        }
        P = act ? P - w : 0u;
        const double* xs = reinterpret_cast<const double*>(slot) + (rec >> 19);
        a_generic<R>(data, P, rec, xs, it_nf, it_gwords, r);
        a_finish<R>(p, r, act, lane, nslot, dest, it_final, cf);
    }
}

// A leaf wider than one chunk: every chunk item writes partial sums, k_reduce
// (launched between the phases) adds them in fixed chunk order.
struct RedCol {
    uint32_t col;      // global column id (C index)
    uint32_t p0;       // partial of chunk 0
    uint32_t stride;   // leaf rank k (partials are chunk-major)
    uint32_t nchunks;
};

// Chunk partials -> c_i = alpha coef_i sum_ch partial.  Columns with many
// chunks (the first nlong entries) take one warp each: lane j adds chunks j,
// j + 32, ... and a fixed butterfly finishes the sum (lane 0's order is the
// same on every run).  The rest take one thread each with independent loads.
constexpr uint32_t kRedLong = 16;  // chunks from which a column gets a warp
template <int R>
__global__ void k_reduce(Params p, const RedCol* rc, uint32_t nlong, uint32_t n) {
    pdl_trigger();
    pdl_wait();  // the partials of phase A
    const uint32_t long_blocks = (nlong + 7) / 8;
    if (blockIdx.x < long_blocks) {
        const uint32_t i = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31u;
        if (i >= nlong) return;
        const RedCol r = rc[i];
        double s0[R], s1[R];  // the R right-hand sides of a chunk are adjacent
#pragma unroll
        for (int c = 0; c < R; ++c) s0[c] = s1[c] = 0.0;
        uint32_t ch = lane;
        for (; ch + 32 < r.nchunks; ch += 64) {
            const double* a0 = p.partial + static_cast<size_t>(r.p0 + ch * r.stride) * R;
            const double* a1 = p.partial + static_cast<size_t>(r.p0 + (ch + 32) * r.stride) * R;
#pragma unroll
            for (int c = 0; c < R; ++c) {
                s0[c] += a0[c];
                s1[c] += a1[c];
            }
        }
        if (ch < r.nchunks) {
            const double* a0 = p.partial + static_cast<size_t>(r.p0 + ch * r.stride) * R;
#pragma unroll
            for (int c = 0; c < R; ++c) s0[c] += a0[c];
        }
        const double cf = p.alpha * p.coef[r.col];
        double* out = rec_c<R>(p, r.col);
#pragma unroll
        for (int c = 0; c < R; ++c) {
            double s = s0[c] + s1[c];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) out[c] = cf * s;
        }
        return;
    }
    const uint32_t i = nlong + (blockIdx.x - long_blocks) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const RedCol r = rc[i];
    constexpr int NC = R == 1 ? 4 : 1;  // independent chains per right-hand side
    double s[R][NC];
#pragma unroll
    for (int c = 0; c < R; ++c)
#pragma unroll
        for (int q = 0; q < NC; ++q) s[c][q] = 0.0;
#pragma unroll
    for (uint32_t ch = 0; ch < kRedLong; ++ch) {
        if (ch < r.nchunks) {
            const double* a0 = p.partial + static_cast<size_t>(r.p0 + ch * r.stride) * R;
#pragma unroll
            for (int c = 0; c < R; ++c) s[c][ch % NC] += a0[c];
        }
    }
    const double cf = p.alpha * p.coef[r.col];
    double* out = rec_c<R>(p, r.col);
#pragma unroll
    for (int c = 0; c < R; ++c) {
        double t = s[c][0];
        if (NC == 4) t = (s[c][0] + s[c][1 % NC]) + (s[c][2 % NC] + s[c][3 % NC]);
        out[c] = cf * t;
    }
}

// ------------------------------------------------------------ phase B ----
// acc[g * R + c]: rows 32 g + lane of the block, right-hand side c.
// generic path: any layout, any row offset / count (lanes individually predicated)
template <int R>
__device__ __forceinline__ void b_column(const uint32_t* seg, uint32_t packed, unsigned w, int f0, unsigned vmask,
                                         unsigned umask, const double (&coef)[R], double (&acc)[kG * R]) {
    const int bit0 = f0 * static_cast<int>(w);
    const uint32_t* sp = seg + (bit0 >> 5);
    const unsigned sh = static_cast<unsigned>(bit0) & 31u;
#pragma unroll
    for (int g = 0; g < kG; ++g) {
        if (umask & (1u << g)) {
            if (vmask & (1u << g)) {
                const double d = dec_generic(sp + g * w, packed, sh);
#pragma unroll
                for (int c = 0; c < R; ++c) acc[g * R + c] = fma(d, coef[c], acc[g * R + c]);
            }
        }
    }
}

template <int R>
__device__ __forceinline__ void b_item_generic(const BItem& it, const uint32_t* seg, const double* cf, unsigned lane,
                                               double dmul, double (&acc)[kG * R]) {
    const unsigned nseg = it.nseg, nr = it.nr;
    // lane owns rows 32 g + lane of the block; field index f0 + 32 g in each segment
    const int f0 = static_cast<int>(lane) - static_cast<int>(it.ra);
    unsigned vmask = 0;
#pragma unroll
    for (int g = 0; g < kG; ++g) {
        const int f = f0 + 32 * g;
        if (f >= 0 && f < static_cast<int>(nr)) vmask |= 1u << g;
    }
    const unsigned umask = __reduce_or_sync(0xffffffffu, vmask);
    const uint8_t* wc = reinterpret_cast<const uint8_t*>(cf);
    for (unsigned c = 0; c < nseg; ++c) {
        const double* rc = reinterpret_cast<const double*>(wc + c * rec_bytes<R>());
        const uint32_t pw = it.kind == 0 ? it.dpacked : reinterpret_cast<const uint32_t*>(rc + R)[2];
        const unsigned w = pw & 0xffu;
        double cc[R];
#pragma unroll
        for (int q = 0; q < R; ++q) cc[q] = it.kind == 0 ? dmul * cf[c * R + q] : rc[q];
        b_column<R>(seg, pw, w, f0, vmask, umask, cc, acc);
        seg += (nr * w + 31) >> 5;
    }
}

// fast path: the item covers row groups [GLO, GHI) of the block completely and
// every column decodes with dec_pair: lane l takes field l + 32 (g - GLO) of
// each column segment, at the same shift in every group.  A segment's NG =
// GHI - GLO groups (32 fields = w words each) are word-interleaved (group g's
// word j at NG j + g): one pair of NG-word vector loads per column.
template <int GLO, int GHI, int R>
__device__ __forceinline__ void b_column_full(const uint32_t* seg, unsigned lane, unsigned w, uint32_t mask,
                                              uint32_t mul, uint64_t bias, const double (&coef)[R],
                                              double (&acc)[kG * R]) {
    constexpr int NG = GHI - GLO;
    const unsigned top = (lane + 1) * w;  // one past the sign bit of field `lane`
    const unsigned s = top;               // the funnel shift takes it modulo 32
    uint32_t lo[NG], hi[NG];
    il_load<NG>(seg, static_cast<int>(top >> 5) - 1, lo, hi);
#pragma unroll
    for (int g = GLO; g < GHI; ++g) {
        const double d = dec_pair(lo[g - GLO], hi[g - GLO], s, mask, mul, bias);
#pragma unroll
        for (int c = 0; c < R; ++c) acc[g * R + c] = fma(d, coef[c], acc[g * R + c]);
    }
}

template <int GLO, int GHI, int R>
__device__ __forceinline__ void b_item_full(const BItem& it, const uint32_t* seg, const double* cf, unsigned lane,
                                            double dmul, uint64_t bias, double (&acc)[kG * R]) {
    const unsigned nseg = it.nseg;
    if (it.kind == 0) {  // dense: one layout for the whole item
        const unsigned w = it.dpacked & 0xffu, e = (it.dpacked >> 16) & 0xffu;
        const uint32_t mask = fast_mask(w), mul = c_pow2e.v[e & 31u];
        const unsigned segw = (GHI - GLO) * w;
        if (R == 1) {
            // sum d * x_c over the item's columns, then one alpha * scale multiply
            double t[kG * R];
#pragma unroll
            for (int g = 0; g < kG * R; ++g) t[g] = 0.0;
#pragma unroll 2
            for (unsigned c = 0; c < nseg; ++c) {
                const double xc[R] = {cf[c]};
                b_column_full<GLO, GHI, R>(seg, lane, w, mask, mul, bias, xc, t);
                seg += segw;
            }
#pragma unroll
            for (int g = GLO; g < GHI; ++g) acc[g] = fma(dmul, t[g], acc[g]);
        } else {
            for (unsigned c = 0; c < nseg; ++c) {
                double xc[R];
#pragma unroll
                for (int q = 0; q < R; ++q) xc[q] = dmul * cf[c * R + q];
                b_column_full<GLO, GHI, R>(seg, lane, w, mask, mul, bias, xc, acc);
                seg += segw;
            }
        }
    } else {
        const uint8_t* wc = reinterpret_cast<const uint8_t*>(cf);  // staged records of the leaf's columns
#pragma unroll 2
        for (unsigned c = 0; c < nseg; ++c) {
            const uint8_t* rp = wc + c * rec_bytes<R>();
            double cc[R];
            uint32_t mask, mul, w;
            if (R == 1) {
                // the record as two 16-byte loads: {c, mask, mul}, {packed, w, -, -}
                const uint4 q0 = reinterpret_cast<const uint4*>(rp)[0];
                const uint4 q1 = reinterpret_cast<const uint4*>(rp)[1];
                cc[0] = __hiloint2double(static_cast<int>(q0.y), static_cast<int>(q0.x));
                mask = q0.z;
                mul = q0.w;
                w = q1.y;
            } else {
#pragma unroll
                for (int q = 0; q < R; ++q) cc[q] = reinterpret_cast<const double*>(rp)[q];
                const uint4 pr = *reinterpret_cast<const uint4*>(rp + 8 * R);  // {mask, mul, packed, w}
                mask = pr.x;
                mul = pr.y;
                w = pr.w;
            }
            b_column_full<GLO, GHI, R>(seg, lane, w, mask, mul, bias, cc, acc);
            seg += (GHI - GLO) * w;
        }
    }
}

// R = 1 bodies (the single-vector product).  Dense: one layout per item; the
// column loop keeps two accumulator sets (even / odd columns) so consecutive
// FMAs on a row do not wait on each other, and one alpha * scale multiply per
// item.  Lowrank W columns: each column's record {c, mask, mul} + w.
template <int GLO, int GHI>
__device__ __forceinline__ void b1_dense(const BItem& it, const uint32_t* seg, const double* xc, unsigned lane,
                                         double dmul, uint64_t bias, double (&acc)[kG]) {
    constexpr int NG = GHI - GLO;
    const unsigned w = it.dpacked & 0xffu, e = (it.dpacked >> 16) & 0xffu;
    const uint32_t mask = fast_mask(w), mul = c_pow2e.v[e & 31u];
    const unsigned top = (lane + 1) * w;                 // one past the sign bit of field `lane`
    const int o = static_cast<int>(top >> 5) - 1;  // same word and shift in every column
    const unsigned s = top;
    const unsigned segw = NG * w;
    double t0[NG], t1[NG];
#pragma unroll
    for (int g = 0; g < NG; ++g) t0[g] = t1[g] = 0.0;
    const unsigned n = it.nseg;
    // pointer induction: the vectors of the CP columns of an iteration (8 fields
    // per lane) sit at fixed offsets from one pointer
    constexpr unsigned CP = 8 / NG;
    seg += static_cast<int>(NG) * o;  // vector o of the first column
    const double* xe = xc + (n & ~(CP - 1u));
    for (; xc != xe; xc += CP) {
        double xv[CP];
        uint32_t l[CP][NG], h[CP][NG];
#pragma unroll
        for (unsigned j = 0; j < CP; ++j) {
            xv[j] = xc[j];
            il_load<NG>(seg + j * segw, 0, l[j], h[j]);
        }
#pragma unroll
        for (int g = 0; g < NG; ++g) {
#pragma unroll
            for (unsigned j = 0; j < CP; j += 2) {
                t0[g] = fma(dec_pair(l[j][g], h[j][g], s, mask, mul, bias), xv[j], t0[g]);
                t1[g] = fma(dec_pair(l[j + 1][g], h[j + 1][g], s, mask, mul, bias), xv[j + 1], t1[g]);
            }
        }
        seg += CP * segw;
    }
    for (unsigned r = n & (CP - 1u); r; --r) {
        const double x0 = *xc++;
        uint32_t l0[NG], h0[NG];
        il_load<NG>(seg, 0, l0, h0);
#pragma unroll
        for (int g = 0; g < NG; ++g) t0[g] = fma(dec_pair(l0[g], h0[g], s, mask, mul, bias), x0, t0[g]);
        seg += segw;
    }
#pragma unroll
    for (int g = 0; g < NG; ++g) acc[GLO + g] = fma(dmul, t0[g] + t1[g], acc[GLO + g]);
}

template <int GLO, int GHI>
__device__ __forceinline__ void b1_lr(const BItem& it, const uint32_t* seg, const uint8_t* rec, unsigned lane,
                                      uint64_t bias, double (&acc)[kG]) {
    constexpr int NG = GHI - GLO;
    const unsigned lp1 = lane + 1;
    const unsigned n = it.nseg;
#pragma unroll (kBLRUnroll * 4 / NG)
    for (unsigned c = 0; c < n; ++c) {
        const uint4 q0 = reinterpret_cast<const uint4*>(rec)[0];  // {c lo, c hi, mask, mul}
        const unsigned w = reinterpret_cast<const uint32_t*>(rec)[5];  // WCol::w
        rec += 32;
        const double cc = __hiloint2double(static_cast<int>(q0.y), static_cast<int>(q0.x));
        const unsigned top = lp1 * w;
        uint32_t lo[NG], hi[NG];
        il_load<NG>(seg, static_cast<int>(word_of(top)) - 1, lo, hi);
#pragma unroll
        for (int g = 0; g < NG; ++g) acc[GLO + g] = fma(dec_pair(lo[g], hi[g], top, q0.z, q0.w, bias), cc, acc[GLO + g]);
        seg += NG * w;
    }
}

template <int R>
__device__ __forceinline__ void b_item(const Params& p, const BItem& it, const uint8_t* slot, unsigned lane,
                                       double (&acc)[kG * R]) {
    if constexpr (R == 1) {
        const double* cf = reinterpret_cast<const double*>(slot + it.coef_off);
        const uint32_t* seg = reinterpret_cast<const uint32_t*>(slot) + it.word_off;
        switch (it.fcase | (it.kind << 2)) {  // one jump table: body x leaf kind
            case 1: b1_dense<0, 4>(it, seg, cf, lane, p.alpha * it.scale, p.bias, acc); return;
            case 2: b1_dense<0, 2>(it, seg, cf, lane, p.alpha * it.scale, p.bias, acc); return;
            case 3: b1_dense<2, 4>(it, seg, cf, lane, p.alpha * it.scale, p.bias, acc); return;
            case 5: b1_lr<0, 4>(it, seg, reinterpret_cast<const uint8_t*>(cf), lane, p.bias, acc); return;
            case 6: b1_lr<0, 2>(it, seg, reinterpret_cast<const uint8_t*>(cf), lane, p.bias, acc); return;
            case 7: b1_lr<2, 4>(it, seg, reinterpret_cast<const uint8_t*>(cf), lane, p.bias, acc); return;
            default: b_item_generic<R>(it, seg, cf, lane, p.alpha * it.scale, acc); return;
        }
    }
    else {
    const double* cf = reinterpret_cast<const double*>(slot + it.coef_off);
    const double dmul = p.alpha * it.scale;  // dense: alpha * buffer scale folded into x
    const uint32_t* seg = reinterpret_cast<const uint32_t*>(slot) + it.word_off;
    // fast bodies for dec_fast layouts at the shapes 64-row leaf clusters
    // produce; everything else takes one generic body (exact for every layout),
    // which keeps the kernel inside the instruction cache
    static_assert(kG == 4, "fast-path table assumes 128-row blocks");
    switch (it.fcase) {  // the body index, precomputed by bcase_of (a dense jump table)
        case 1: b_item_full<0, 4, R>(it, seg, cf, lane, dmul, p.bias, acc); break;
        case 2: b_item_full<0, 2, R>(it, seg, cf, lane, dmul, p.bias, acc); break;
        case 3: b_item_full<2, 4, R>(it, seg, cf, lane, dmul, p.bias, acc); break;
        default:
            b_item_generic<R>(it, seg, cf, lane, dmul, acc);  // also uncompressed words (modes 3-5)
            break;
    }
    }
}

template <int NW>
__device__ __forceinline__ void consumer_bar() {  // the consumer warps of phase B only
    asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");
}

// Persistent kernels: one CTA per resident slot, stripes claimed dynamically.
template <int R>
__global__ void __launch_bounds__(kThreadsA, kCtasA) k_phase_a(Params p) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kRingBytesA);
    uint64_t* empty = full + kNStageA;
    Mail* mail = reinterpret_cast<Mail*>(empty + kNStageA);
    const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    // phase B's stripe counter for this product (A runs first, B claims only
    // after its griddepcontrol.wait, so the store is visible by then)
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        p.work[1] = 0u;
        __threadfence();  // visible before this CTA triggers phase B's launch
    }
    ring_init<kNWA, kNStageA>(full, empty, mail);
    pdl_trigger();
    if (warp == kNWA) {
        producer<true, R>(p, smem, full, empty, mail, lane);
        return;
    }
    if (warp > kNWA) {
        coef_producer<true, R>(p, smem, full, empty, mail, lane);
        return;
    }
    consume<kNWA, true>(
        smem, full, empty, warp, lane, dbg(p),
        [&](const uint8_t* base, unsigned i) {
            a_item<R>(p, reinterpret_cast<const AItem*>(base) + i, base, lane);
        },
        [](uint32_t) {});
}

template <int R>
__global__ void __launch_bounds__((nwb<R>() + kNProd) * 32, kCtasB) k_phase_b(Params p) {
    constexpr int NW = nwb<R>();
    extern __shared__ __align__(128) uint8_t smem[];
    double* red = reinterpret_cast<double*>(smem + kRingBytes);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kRingBytes + kRedBytes);
    uint64_t* empty = full + kNStage;
    Mail* mail = reinterpret_cast<Mail*>(empty + kNStage);
    const unsigned tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    ring_init<NW, kNStage>(full, empty, mail);
    if (warp == NW) {
        producer<false, R>(p, smem, full, empty, mail, lane);
        return;
    }
    if (warp > NW) {
        coef_producer<false, R>(p, smem, full, empty, mail, lane);
        return;
    }
    double acc[kG * R];
#pragma unroll
    for (int g = 0; g < kG * R; ++g) acc[g] = 0.0;
    constexpr unsigned H = NW / 2;
    static_assert(NW % 2 == 0, "phase B's pairwise warp reduction needs an even number of consumer warps");
    static_assert(H * kR * sizeof(double) <= kRedBytes, "phase-B reduction buffer");
    consume<NW, false>(
        smem, full, empty, warp, lane, dbg(p),
        [&](const uint8_t* base, unsigned i) {
            b_item<R>(p, reinterpret_cast<const BItem*>(base + kRangeBytes)[i], base, lane, acc);
        },
        [&](uint32_t sid) {  // block done: fixed-order pairwise sum of the warps, then y
            const uint4 sr = p.stripe_b[sid];
            const uint32_t blk = sr.z, piece = sr.w;
            const uint32_t r0 = p.row_begin + blk * kR;
            const uint32_t nrows = min(static_cast<uint32_t>(kR), p.row_end - r0);
#pragma unroll
            for (int c = 0; c < R; ++c) {  // one right-hand side at a time through the buffer
                consumer_bar<NW>();
                if (warp >= H) {
#pragma unroll
                    for (int g = 0; g < kG; ++g) red[(warp - H) * kR + 32 * g + lane] = acc[g * R + c];
                }
                consumer_bar<NW>();
                if (warp < H) {
#pragma unroll
                    for (int g = 0; g < kG; ++g) acc[g * R + c] += red[warp * kR + 32 * g + lane];
                }
                consumer_bar<NW>();
                if (warp < H) {
#pragma unroll
                    for (int g = 0; g < kG; ++g) red[warp * kR + 32 * g + lane] = acc[g * R + c];
                }
                consumer_bar<NW>();
                if (tid < nrows) {
                    double sum = 0.0;
#pragma unroll
                    for (unsigned wv = 0; wv < H; ++wv) sum += red[wv * kR + tid];
                    if (piece == 0) {
                        double* yp = p.y + static_cast<size_t>(r0 + tid) * R + c;
                        *yp = p.beta == 0.0 ? sum : fma(p.beta, *yp, sum);
                    } else {  // one part of a split block: k_combine adds the parts and beta y
                        const size_t nl = p.row_end - p.row_begin;
                        p.ypart[((piece - 1) * nl + (r0 - p.row_begin + tid)) * R + c] = sum;
                    }
                }
            }
            consumer_bar<NW>();
#pragma unroll
            for (int g = 0; g < kG * R; ++g) acc[g] = 0.0;
        });
}

// Row blocks split into pieces (few blocks per GPU, e.g. one rank of a block-row
// partition): y = beta y + sum of the pieces' partial sums, in piece order.
template <int R>
__global__ void k_combine(Params p, const uint8_t* npieces) {
    pdl_trigger();
    pdl_wait();  // phase B's partial sums
    const size_t nl = p.row_end - p.row_begin;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < nl * R;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t row = i / R;
        const unsigned q = npieces[row / kR];
        if (q == 0) continue;
        double sum = 0.0;
        for (unsigned j = 0; j < q; ++j) sum += p.ypart[j * nl * R + i];
        double* yp = p.y + p.row_begin * static_cast<size_t>(R) + i;
        *yp = p.beta == 0.0 ? sum : fma(p.beta, *yp, sum);
    }
}

// ---------------------------------------------------- complex arenas ----
// A = U S V^H with U = Ur + i Ui, V = Vr + i Vi held as W = [Ur Ui], X = [Vr Vi]
// (hcmx_hmat_desc::complex_pairs); x and y interleave two complex columns,
// [Re x1, Im x1, Re x2, Im x2].  V^H x = (Vr^T Re x + Vi^T Im x) + i (Vr^T Im x -
// Vi^T Re x): phase A leaves a = alpha s_Vr Vr'^T x4 and b = alpha s_Vi Vi'^T x4
// in the records of the pair's two X columns; k_ccombine forms t = V^H x and
// writes the W columns' coefficients, Ur_j: s_Ur sigma (t_r, t_i), Ui_j:
// s_Ui sigma (-t_i, t_r), so phase B's real accumulation gives Re / Im y.  The
// imaginary dense parts read the swapped x (-Im x, Re x) (copy table 2).
struct CPair {
    uint32_t a, b;  // record (rank column) of Ur_j / Vr_j and of Ui_j / Vi_j
    double sig, sa, sb;
};
static_assert(sizeof(CPair) == 32, "CPair layout");

// x: n x R row-major, R / 2 complex columns interleaved (Re, Im): each (Re, Im)
// pair becomes (-Im, Re)
__global__ void k_xswap(const double* __restrict__ x, double* __restrict__ x2, uint64_t npairs) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < npairs; i += gridDim.x * (uint64_t)blockDim.x) {
        const double2 u = reinterpret_cast<const double2*>(x)[i];
        reinterpret_cast<double2*>(x2)[i] = make_double2(-u.y, u.x);
    }
}

template <int R>
__global__ void k_ccombine(Params p, const CPair* __restrict__ cp, uint32_t n) {
    pdl_trigger();
    pdl_wait();  // phase A (and k_reduce) wrote the X^T x halves
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const CPair q = cp[i];
        double* ra = rec_c<R>(p, q.a);
        double* rb = rec_c<R>(p, q.b);
#pragma unroll
        for (int c = 0; c < R; c += 2) {  // complex column c / 2
            const double tr = q.sig * (ra[c] + rb[c + 1]), ti = q.sig * (ra[c + 1] - rb[c]);
            ra[c] = q.sa * tr, ra[c + 1] = q.sa * ti;
            rb[c] = -q.sb * ti, rb[c + 1] = q.sb * tr;
        }
    }
}

__global__ void k_scale(double* y, uint64_t n, double beta) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += gridDim.x * (uint64_t)blockDim.x)
        y[i] = beta == 0.0 ? 0.0 : beta * y[i];
}

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
    // phase-A items (gwords > 0): field j in row j % kARows of group j / kARows
    // at bit pbit of the row, the row's words kARows apart from `word` +
    // (j / kARows) gwords + j % kARows; phase-B segments with il > 1: il
    // word-interleaved groups of 32 fields (field j at bit (j % 32) w of group
    // j / 32, whose words are il apart from `word` + j / 32); else contiguous
    uint32_t pbit;
    uint16_t rowbits, gwords;
    uint8_t il = 0;
};

// field locator of a SegRef: the word-strided stream (first word, stride) and bit of field j
struct FieldLoc {
    uint64_t word;
    unsigned stride;
    uint64_t bit;
};
inline FieldLoc field_loc(const SegRef& r, uint64_t j, unsigned w) {
    if (r.gwords) return {(j / kARows) * r.gwords + (j % kARows), static_cast<unsigned>(kARows), r.pbit};
    if (r.il > 1) return {j / 32, r.il, (j % 32) * w};
    return {0, 1u, j * w};
}

// w (<= 64) bits at bit offset `bit` of the LSB-first stream src[0, len)
// (bytes past len read as 0)
uint64_t get_bits(const uint8_t* src, uint64_t len, uint64_t bit, unsigned w) {
    const uint64_t byte = bit >> 3;
    uint8_t tmp[16] = {};
    if (byte + 16 <= len) std::memcpy(tmp, src + byte, 16);
    else if (byte < len) std::memcpy(tmp, src + byte, static_cast<size_t>(len - byte));
    unsigned __int128 v;
    std::memcpy(&v, tmp, 16);
    const uint64_t r = static_cast<uint64_t>(v >> (bit & 7));
    return w >= 64 ? r : (r & ((1ull << w) - 1));
}

// OR the low w bits of v into the word stream dst at bit offset `bit` (the
// stream's words `stride` apart)
void put_bits(uint32_t* dst, uint64_t bit, uint64_t v, unsigned w, unsigned stride = 1) {
    while (w) {
        const unsigned sh = static_cast<unsigned>(bit & 31), take = std::min(32u - sh, w);
        const uint64_t part = take == 64 ? v : (v & ((1ull << take) - 1));
        dst[(bit >> 5) * stride] |= static_cast<uint32_t>(part << sh);
        v = take >= 64 ? 0 : v >> take;
        bit += take;
        w -= take;
    }
}

// w (<= 64) bits at bit offset `bit` of a word stream whose words are `stride`
// apart (words past nwords read as 0)
uint64_t get_bits_strided(const uint32_t* src, uint64_t nwords, unsigned stride, uint64_t bit, unsigned w) {
    unsigned __int128 v = 0;
    const uint64_t k0 = bit >> 5;
    for (unsigned t = 0; t < 3; ++t) {
        const uint64_t idx = (k0 + t) * stride;
        if (idx < nwords) v |= static_cast<unsigned __int128>(src[idx]) << (32 * t);
    }
    const uint64_t r = static_cast<uint64_t>(v >> (bit & 31));
    return w >= 64 ? r : (r & ((1ull << w) - 1));
}

// one lane of a phase-A item: fields [f0, f0 + nf) of codec buffer `buf`
// (a chunk of one X column), x elements [xidx, xidx + nf).  Lanes come in
// segments of G (a power of two) chunks of one rank column, summed in-warp
// into result element `dest` (wcol record if final_, else a partial); g is
// the lane's place in its segment.
struct ALane {
    uint64_t buf, f0;
    uint32_t nf, xidx, dest, final_, G, g;
};

}  // namespace
}  // namespace hcmx_gpu

using namespace hcmx_gpu;

struct hcmx_hmat {
    uint64_t n_rows = 0, n_cols = 0, rb = 0, re = 0;
    int R = 1;                   // right-hand sides per product of this arena (1 or kMultiR)
    DevBuf arena, stages, stripe_a, stripe_b, copies, work, wcol, coef, partial,
        redcols, xpad, xbuf, ybuf;
    uint32_t nstripe_a = 0, nblocks = 0, nlr = 0, nred = 0, nred_long = 0, pieces = 0;
    DevBuf npieces, ypart;  // split row blocks (pieces > 0): pieces per block, partial row sums
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
    hcmx_hmat* trans = nullptr;  // M^T (hmatrix.hpp:128 transpose), built on request
    hcmx_hmat* multi = nullptr;  // the same matrix laid out for kMultiR right-hand sides (matmat)
    bool cplx = false;           // complex arena (hcmx_hmat_desc::complex_pairs; R = kMultiR)
    DevBuf xswap, cpairs;        // complex: swapped x (n x 4), rank-pair table for k_ccombine
    uint32_t ncpairs = 0;
    // products on one handle share its device scratch (stripe counters, x copy,
    // phase-A results): a product issued on another stream than the previous
    // one first waits for it (the reference's matvec is re-entrant, const M&)
    std::mutex mu, io_mu;  // io_mu: the host-pointer calls' staging buffers (xbuf / ybuf)
    cudaEvent_t last = nullptr;
    cudaStream_t last_stream = nullptr;
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

// host-side column parameters of the decoders (dec_fast / dec_generic)
ColPar col_par(const hcmx_descriptor& x) {
    ColPar c{};
    const unsigned w = x.bit_width, m = x.mant_bits, e = x.exp_bits;
    unsigned mode = (w > 32 || e >= 11 || w != 1 + e + m) ? 2u : 0u;
    if (x.scheme >= HCMX_RAW_F64) mode = 3u + (x.scheme - HCMX_RAW_F64);  // uncompressed storage
    if (mode == 0) {
        c.mask = ((1u << (w - 1)) - 1u) << (32 - w);
        c.mul = 1u << (21 + e);
    }
    c.packed = w | (m << 8) | (e << 16) | (mode << 24);
    c.w = w;
    return c;
}

// fast-path case of a phase-B item covering rows [ra, ra + nr) of its block
uint8_t fcase_of(uint64_t ra, uint64_t nr) {
    if (ra % 32 || nr % 32) return 0;
    const unsigned lo = static_cast<unsigned>(ra / 32), hi = static_cast<unsigned>((ra + nr) / 32);
    const unsigned c = lo << 4 | hi;
    switch (c) {
        case 0x04: case 0x02: case 0x24: return static_cast<uint8_t>(c);
        default: return 0;
    }
}

// phase-B body index: whole row groups [0,4) / [0,2) / [2,4) with the fast decoder
uint8_t bcase_of(uint64_t ra, uint64_t nr, unsigned mode) {
    const uint8_t f = fcase_of(ra, nr);
    if (mode != 0 || f == 0) return 0;
    return static_cast<uint8_t>(f == 0x04 ? 1 : f == 0x02 ? 2 : 3);
}

inline uint32_t r16(uint64_t x) { return static_cast<uint32_t>((x + 15) & ~uint64_t(15)); }

// A run of fields of one codec buffer that an item needs (copied word aligned)
struct Seg {
    uint64_t buf, f0, nf;
};

// An item before placement: descriptor + the field runs it streams
template <class Item>
struct Spec {
    Item it;
    uint32_t seg0, nseg;   // range in Builder::segs
    uint64_t words;        // packed words
    uint32_t coef_x;       // A: x slice bytes (shareable by the chunk's items)
    uint32_t coef_p;       // coefficient / params bytes owned by the item
    uint64_t cost;         // fields (LPT weight)
    uint64_t unit;         // item key: consecutive columns with the same key may merge
    uint32_t xidx, nf;     // A: x slice key
    uint32_t param;        // lowrank / phase A: packed column layout stored ahead of the segments
    uint32_t elem;         // this column's coefficient index (x or C)
    uint32_t sl_table, sl_start, sl_count;  // staged coefficient slice (deduplicated per stage)
};

// split columns [0, n) into consecutive groups of <= maxcols columns and,
// beyond the first column, <= kItemTarget packed bytes
template <class WordsOf>
std::vector<std::pair<uint32_t, uint32_t>> column_groups(uint32_t n, uint32_t maxcols, WordsOf words_of) {
    std::vector<std::pair<uint32_t, uint32_t>> g;
    uint32_t c0 = 0;
    while (c0 < n) {
        uint32_t c1 = c0 + 1;
        uint64_t bytes = words_of(c0) * 4;
        while (c1 < n && c1 - c0 < maxcols && bytes + words_of(c1) * 4 <= kItemTarget) bytes += words_of(c1++) * 4;
        g.emplace_back(c0, c1 - c0);
        c0 = c1;
    }
    return g;
}

// word interleave of a phase-B item's column segments: the fast bodies read
// NG = 4 (rows [0,128)) or 2 (rows [0,64) / [64,128)) interleaved groups per
// column; generic items keep each segment's fields contiguous
inline unsigned il_of(const BItem& it) { return it.fcase == 1 ? 4u : (it.fcase == 2 || it.fcase == 3) ? 2u : 1u; }
template <class Item>
inline unsigned il_of(const Item&) { return 1u; }

// anonymous, lazily backed host mapping (pages cost nothing until written)
struct HostBlob {
    uint8_t* p = nullptr;
    size_t bytes = 0;
    void map(size_t n) {
        bytes = std::max<size_t>(n, 1);
        void* q = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
        if (q == MAP_FAILED) throw oom_error("hmat: host mapping of the blob failed");
        p = static_cast<uint8_t*>(q);
    }
    ~HostBlob() {
        if (p) munmap(p, bytes);
    }
};

struct Builder {
    const hcmx_hmat_desc& d;
    hcmx_hmat* h;
    const uint8_t* blob = nullptr;
    bool keep_map = false;

    std::vector<uint32_t> arena;  // words
    std::vector<Stage> stages;
    std::vector<BItem> bitems;
    std::vector<Seg> segs;
    std::vector<uint64_t> copies;  // kCopies per stage

    static uint64_t copy_entry(uint32_t idx, uint32_t dst, uint32_t bytes, unsigned table) {
        return (1ull << 63) | (static_cast<uint64_t>(table) << 60) | (static_cast<uint64_t>(bytes / 16) << 48) |
               (static_cast<uint64_t>(dst / 16) << 32) | idx;
    }

    int R = 1;  // right-hand sides: x / coefficient elements are R doubles wide

    Builder(const hcmx_hmat_desc& dd, hcmx_hmat* hh) : d(dd), h(hh), R(hh->R) {}

    // the bytes a stage's copies deliver must be exactly what its full barrier
    // expects, or the consumers would wait forever
    void check_copies(size_t c0, uint32_t expect) const {
        uint64_t sum = 0;
        for (size_t q = c0; q < c0 + kCopies; ++q)
            if (copies[q] >> 63) sum += ((copies[q] >> 48) & 0xfffu) * 16u;
        if (sum != expect) throw std::logic_error("hmat: stage copy bytes mismatch");
    }

    unsigned width(uint64_t b) const { return d.desc[b].bit_width; }
    uint64_t words_of(uint64_t b, uint64_t nf) const { return (nf * width(b) + 31) / 32; }

    // The layout pass only sizes the arena and records where every field run
    // goes; the bits are placed afterwards by place_all() on all host cores
    // (item / segment destinations are disjoint word ranges).
    struct CopyJob {   // phase B: fields [f0, f0+nf) of buffer buf, word aligned at arena word `at`
        uint64_t at, buf, f0, nf;
        unsigned il;    // > 1: il groups of 32 fields, word-interleaved (fast-body segments)
    };
    struct LaneJob {   // phase A: one lane of an item (row-interleaved placement)
        uint64_t data0, buf, f0;
        uint32_t nf, P, rowbits, gwords;
    };
    std::vector<CopyJob> copy_jobs;
    std::vector<LaneJob> lane_jobs;

    // append the words of fields [f0, f0+nf) of buffer b (word aligned); il >
    // 1: nf = 32 il fields as il word-interleaved groups (group g's word j at
    // il j + g, the layout of the phase-B fast bodies)
    void put_fields(const Seg& s, unsigned il = 1) {
        const unsigned w = width(s.buf);
        const uint64_t nw = (s.nf * w + 31) / 32;
        if (il > 1 && s.nf != 32ull * il) throw std::logic_error("hmat: interleaved segment");
        const uint64_t at = arena.size();
        arena.resize(at + nw);
        copy_jobs.push_back({at, s.buf, s.f0, s.nf, il});
        if (keep_map) {
            SegRef r{at, static_cast<uint32_t>(s.f0), static_cast<uint32_t>(s.nf), 0, 0, 0};
            r.il = static_cast<uint8_t>(il);
            h->segs[s.buf].push_back(r);
        }
    }

    void place_all() {
        unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
        const size_t nc = copy_jobs.size(), nl = lane_jobs.size();
        auto work = [&](unsigned t) {
            uint32_t tmp[64];
            for (size_t i = t; i < nc; i += nt) {
                const CopyJob& j = copy_jobs[i];
                const unsigned w = width(j.buf);
                if (j.il <= 1) {
                    copy_bits(blob + d.poff[j.buf], static_cast<uint64_t>(d.plen[j.buf]), j.f0 * w, j.nf * w,
                              arena.data() + j.at);
                    continue;
                }
                for (unsigned g = 0; g < j.il; ++g) {  // group g: w words, scattered il apart
                    copy_bits(blob + d.poff[j.buf], static_cast<uint64_t>(d.plen[j.buf]), (j.f0 + 32ull * g) * w,
                              32ull * w, tmp);
                    for (unsigned q = 0; q < w; ++q) arena[j.at + static_cast<uint64_t>(q) * j.il + g] = tmp[q];
                }
            }
            // lanes of one item share words: an item's lanes are consecutive in
            // lane_jobs and go to the same thread (chunks cut at item starts)
            const size_t per = (nl + nt - 1) / nt;
            size_t a = std::min(nl, per * t), b = std::min(nl, per * (t + 1));
            auto item_start = [&](size_t i) {
                while (i > 0 && i < nl && lane_jobs[i].data0 == lane_jobs[i - 1].data0) ++i;
                return i;
            };
            a = item_start(a);
            b = item_start(b);
            for (size_t i = a; i < b; ++i) {
                const LaneJob& L = lane_jobs[i];
                const unsigned w = width(L.buf);
                const uint8_t* src = blob + d.poff[L.buf];
                const uint64_t len = static_cast<uint64_t>(d.plen[L.buf]);
                for (uint32_t q = 0; q < L.nf; ++q) {
                    const uint64_t v = get_bits(src, len, (L.f0 + q) * w, w);
                    // row q % kARows of group q / kARows: its words kARows apart
                    put_bits(arena.data() + L.data0 + static_cast<uint64_t>(q / kARows) * L.gwords + q % kARows, L.P, v,
                             w, kARows);
                }
            }
        };
        std::vector<std::thread> pool;
        for (unsigned t = 1; t < nt; ++t) pool.emplace_back(work, t);
        work(0);
        for (auto& th : pool) th.join();
        copy_jobs.clear();
        lane_jobs.clear();
    }

    // One CTA stripe.  Specs are single columns.  Stages take columns in order
    // up to kStageBytes; consecutive columns of one leaf / row range (B) or leaf
    // chunk (A) with one decode mode merge into items of <= MAXC columns and
    // <= kItemMaxBytes.  Consumer warps claim a stage's items one at a time
    // (largest first), so no per-warp shares are precomputed.  Items of one
    // stage share deduplicated coefficient slices (x or phase-A results).
    template <class Item, int MAXC, int NW>
    void emit_stripe(std::vector<Spec<Item>>& specs, std::vector<Item>& items) {
        size_t pos = 0;
        while (pos < specs.size()) {
            // columns of this stage by data budget
            size_t end = pos;
            uint64_t bytes = 0;
            while (end < specs.size() && bytes + specs[end].words * 4 <= static_cast<uint64_t>(kStageBytes))
                bytes += specs[end++].words * 4;
            if (end == pos) throw invalid_argument("hmat: column exceeds a stage");
            for (;;) {
                if (try_stage<Item, MAXC, NW>(specs, pos, end, items)) break;
                end = pos + std::max<size_t>(1, (end - pos) * 3 / 4);  // too many items / coefficients
            }
            pos = end;
        }
    }

    // items for specs[pos, end); false (nothing emitted) if over budget.
    // NW == 0: items claimed dynamically, largest first.  NW > 0: the stage's
    // columns are cut into NW contiguous pieces of (nearly) equal decode cost,
    // one per consumer warp, and items never straddle a piece.
    template <class Item, int MAXC, int NW>
    bool try_stage(std::vector<Spec<Item>>& specs, size_t pos, size_t end, std::vector<Item>& items) {
        constexpr bool IS_A = std::is_same<Item, AItem>::value;
        struct Built {
            Item it;
            size_t first, n;
            uint64_t words;
        };
        std::vector<Built> built;
        // Coefficient ranges the stage's items read (table 0: x, 8-byte entries,
        // copied from an even index; table 1: WCol records).  Ranges of one table
        // that overlap or lie close together merge into one bulk copy: each copy
        // costs the producer far more than the few extra bytes it brings.
        struct Slice {
            uint32_t table, start, end, off;  // [start, end) elements; start even for table 0
        };
        std::vector<Slice> slices;
        uint32_t coef = 0, data_bytes = 0;
        auto esize = [&](uint32_t table) { return table == 1 ? rec_bytes_rt(R) : 8u * R; };  // 0 x, 2 swapped x: R doubles
        auto slice_bytes = [&](const Slice& s) { return r16((s.end - s.start) * esize(s.table)); };
        std::vector<size_t> cut = {pos, end};
        if (NW > 0) {
            uint64_t total = 0;
            for (size_t i = pos; i < end; ++i) total += specs[i].cost;
            cut.assign(NW + 1, end);
            cut[0] = pos;
            size_t i = pos;
            uint64_t acc = 0;
            for (int q = 1; q < NW; ++q) {
                const uint64_t target = total * q / NW;
                while (i < end && acc + specs[i].cost / 2 <= target) acc += specs[i++].cost;
                cut[q] = i;
            }
        }
        std::vector<uint32_t> piece_end;  // items per piece, cumulative
        for (size_t q = 0; q + 1 < cut.size(); ++q) {
          size_t i = cut[q];
          const size_t pend = cut[q + 1];
          while (i < pend) {
            size_t j = i + 1;
            uint64_t words = specs[i].words;
            while (j < pend && j - i < static_cast<size_t>(MAXC) && specs[j].unit == specs[i].unit &&
                   (words + specs[j].words) * 4 <= kItemMaxBytes)
                words += specs[j++].words;
            Item it = specs[i].it;
            it.nseg = static_cast<uint8_t>(j - i);
            const uint32_t t = specs[i].sl_table;
            slices.push_back({t, t != 1 ? specs[i].sl_start & ~1u : specs[i].sl_start,
                              specs[i].sl_start + specs[i].sl_count, 0});
            built.push_back({it, i, j - i, words});
            i = j;
          }
          piece_end.push_back(static_cast<uint32_t>(built.size()));
        }
        {  // merge: sort by (table, start); join ranges whose gap is small
            std::sort(slices.begin(), slices.end(), [](const Slice& a, const Slice& b) {
                return a.table != b.table ? a.table < b.table : a.start < b.start;
            });
            std::vector<Slice> merged;
            for (const Slice& s : slices) {
                const uint32_t gap = s.table != 1 ? 32u : 4u;  // elements (256 B of x, 128 B of records)
                if (!merged.empty() && merged.back().table == s.table && s.start <= merged.back().end + gap) {
                    merged.back().end = std::max(merged.back().end, s.end);
                } else {
                    merged.push_back(s);
                }
            }
            slices.swap(merged);
            // the coefficients follow the stage in the slot (slot-relative offsets)
            size_t data_words = (built.size() * (kItemBytes / 4) + (NW > 0 ? kRangeBytes / 4 : 0) + 3) & ~size_t(3);
            for (const Built& b : built) data_words = ((data_words + il_of(b.it) - 1) & ~size_t(il_of(b.it) - 1)) + b.words;
            data_bytes = static_cast<uint32_t>(((data_words + 3) & ~size_t(3)) * 4);
            coef = data_bytes;
            for (Slice& s : slices) {
                s.off = coef;
                coef += slice_bytes(s);
            }
            for (Built& b : built) {  // item offsets into the merged ranges
                const Spec<Item>& sp = specs[b.first];
                const uint32_t t = sp.sl_table;
                for (const Slice& s : slices) {
                    if (s.table == t && s.start <= sp.sl_start && sp.sl_start + sp.sl_count <= s.end) {
                        const uint32_t off = s.off + (sp.elem - s.start) * esize(t);
                        if constexpr (IS_A) b.it.x_off = off;
                        else b.it.coef_off = off;
                        break;
                    }
                }
            }
        }
        if (built.size() > static_cast<size_t>(kMaxItems) || coef > static_cast<uint32_t>(kSlotData) ||
            slices.size() > static_cast<size_t>(kCopies)) {
            if (end - pos == 1) throw invalid_argument("hmat: column exceeds a stage");
            return false;
        }
        if (NW == 0)  // claimed largest first: the last items to finish are the small ones
            std::stable_sort(built.begin(), built.end(),
                             [](const Built& x, const Built& y) { return x.words > y.words; });
        static_assert(NW <= kRangeBytes / 4, "phase-B warp ranges");
        uint32_t ranges[kRangeBytes / 4] = {};
        if (NW > 0) {
            uint32_t b0 = 0;
            for (size_t q = 0; q < kRangeBytes / 4; ++q) {
                const uint32_t e = q < piece_end.size() ? piece_end[q] : static_cast<uint32_t>(built.size());
                ranges[q] = b0 | (e << 16);
                b0 = e;
            }
        }
        const size_t c0 = copies.size();
        copies.resize(c0 + kCopies, 0);
        for (size_t q = 0; q < slices.size(); ++q)
            copies[c0 + q] = copy_entry(slices[q].start, slices[q].off, slice_bytes(slices[q]), slices[q].table);
        while (arena.size() % 4) arena.push_back(0u);  // 16-byte aligned stages
        const uint64_t start = arena.size();
        Stage st{};
        st.item0 = static_cast<uint32_t>(items.size());
        // [items][warp ranges (B)][data]: item word offsets count from the stage start
        const size_t head_words = NW > 0 ? kRangeBytes / 4 : 0;  // [warp ranges][items]
        const size_t meta_words = built.size() * (kItemBytes / 4) + head_words;
        arena.resize(start + ((meta_words + 3) & ~size_t(3)), 0u);
        for (Built& b : built) {
            const unsigned il = il_of(b.it);  // interleaved segments: il-word aligned item data
            while ((arena.size() - start) % il) arena.push_back(0u);
            b.it.word_off = static_cast<uint32_t>(arena.size() - start);
            if (IS_A)  // packed column layouts ahead of the segments
                for (size_t k = b.first; k < b.first + b.n; ++k) arena.push_back(specs[k].param);
            for (size_t k = b.first; k < b.first + b.n; ++k)
                for (uint32_t q = 0; q < specs[k].nseg; ++q) put_fields(segs[specs[k].seg0 + q], il);
            items.push_back(b.it);
        }
        for (size_t i = 0; i < built.size(); ++i)
            std::memcpy(arena.data() + start + head_words + i * (kItemBytes / 4), &built[i].it, kItemBytes);
        if (NW > 0) std::memcpy(arena.data() + start, ranges, kRangeBytes);
        while (arena.size() % 4) arena.push_back(0u);
        st.byte_off = start * 4;
        st.bytes = static_cast<uint32_t>((arena.size() - start) * 4);
        st.nitems = static_cast<uint32_t>(built.size());
        // estimated consumer cost (warp instructions): per item, per column, per field
        uint64_t cost = 0;
        for (const Built& b : built) {
            cost += 100;
            for (size_t k = b.first; k < b.first + b.n; ++k) {
                uint64_t fields = 0;
                for (uint32_t q = 0; q < specs[k].nseg; ++q) fields += segs[specs[k].seg0 + q].nf;
                cost += 15 + 12 * ((fields + 31) / 32);
            }
        }
        st.pad = cost;
        if (st.bytes != data_bytes) throw std::logic_error("hmat: stage size");
        st.coef_bytes = coef - data_bytes;
        check_copies(c0, st.coef_bytes);
        stages.push_back(st);
        return true;
    }

    // ---- phase A --------------------------------------------------------
    uint64_t a_items = 0;

    struct AIt {
        size_t l0, nl;
        uint32_t rowbits, gwords, ngroups;
        uint64_t bytes;  // lane records + data, 16-byte aligned
    };

    // A stripe's lanes -> items (<= kALanes lanes with one row count, one
    // result kind and consecutive result elements, <= kAItemBytes of data) ->
    // stages.
    void emit_stripe_a(const std::vector<ALane>& lanes) {
        std::vector<AIt> its;
        for (size_t i = 0; i < lanes.size();) {
            // whole segments only; one row count, result kind and segment size;
            // consecutive results
            // the x slices the item needs must fit one stage's coefficient area
            uint32_t rb = 0, xbytes = 0, nslices = 0;
            size_t j = i;
            while (j < lanes.size()) {
                const ALane& L = lanes[j];
                const size_t seg = L.G;
                if (j + seg - i > static_cast<size_t>(kALanes)) break;
                if (j > i && (L.nf != lanes[i].nf || L.final_ != lanes[i].final_ || L.G != lanes[i].G ||
                              L.dest != lanes[j - 1].dest + 1))
                    break;
                uint32_t sb = 0, xb = 0, ns = 0;
                for (size_t q = j; q < j + seg; ++q) {
                    sb += width(lanes[q].buf);
                    bool seen = false;  // x slice already counted for this item
                    for (size_t u = i; u < q && !seen; ++u) seen = lanes[u].xidx == lanes[q].xidx && lanes[u].nf == lanes[q].nf;
                    if (!seen) {
                        xb += r16((lanes[q].nf + 2) * 8ull * R);
                        ++ns;
                    }
                }
                if (j > i && (static_cast<uint64_t>(rb + sb) * L.nf > 8 * kAItemBytes ||
                              xbytes + xb > kAItemXBytes || nslices + ns > static_cast<uint32_t>(kCopies)))
                    break;
                rb += sb;
                xbytes += xb;
                nslices += ns;
                j += seg;
            }
            AIt t{};
            t.l0 = i;
            t.nl = j - i;
            t.rowbits = rb;
            t.gwords = kARows * ((rb + 31) / 32);  // rows padded to words, word-interleaved
            t.ngroups = (lanes[i].nf + kARows - 1) / kARows;
            const size_t nrec = lanes[i].G == 1 ? t.nl : static_cast<size_t>(kALanes);  // lane records
            t.bytes = r16(4 * (((nrec + 3) & ~size_t(3)) + static_cast<uint64_t>(t.ngroups) * t.gwords));
            if (rb >= (1u << 16) || t.gwords >= (1u << 16)) throw invalid_argument("hmat: phase-A item too wide");
            its.push_back(t);
            i = j;
        }
        for (size_t pos = 0; pos < its.size();) {
            size_t end = pos;
            uint64_t bytes = 0;
            while (end < its.size() && end - pos < static_cast<size_t>(kMaxItems) &&
                   bytes + its[end].bytes + kItemBytes * (end - pos + 1) <= static_cast<uint64_t>(kStageMaxA))
                bytes += its[end++].bytes;
            if (end == pos) throw invalid_argument("hmat: phase-A item exceeds a stage");
            while (!try_stage_a(lanes, its, pos, end)) {  // too many x slices: one item fewer
                if (end - pos == 1) throw invalid_argument("hmat: phase-A item exceeds a stage");
                --end;
            }
            pos = end;
        }
    }

    bool try_stage_a(const std::vector<ALane>& lanes, std::vector<AIt>& its, size_t pos, size_t end) {
        // x slices of the stage's lanes, merged like phase B's coefficient ranges
        // Lanes of a chunk segment (G > 1) read G different x chunks in the same
        // step: each chunk gets its own slice, 16 bytes apart modulo 128, so
        // their LDS.128 hit different banks (merged ranges would put them 512 B
        // apart: one bank group).  Other slices merge as in phase B.
        struct Slice {
            uint32_t start, end, off, pad;
        };
        std::vector<Slice> sl;
        for (size_t t = pos; t < end; ++t)
            for (size_t q = its[t].l0; q < its[t].l0 + its[t].nl; ++q) {
                const ALane& L = lanes[q];
                const uint32_t pad = L.G > 1 ? 1u : 0u;
                const Slice x{pad ? L.xidx : (L.xidx & ~1u), L.xidx + L.nf, 0, pad};
                bool dup = false;
                for (size_t u = sl.size(); u-- > 0 && !dup && sl.size() - u <= 8;)
                    dup = sl[u].start == x.start && sl[u].end == x.end && sl[u].pad == x.pad;
                if (!dup) sl.push_back(x);
            }
        std::sort(sl.begin(), sl.end(), [](const Slice& a2, const Slice& b2) {
            return a2.start != b2.start ? a2.start < b2.start : a2.pad < b2.pad;
        });
        std::vector<Slice> merged;
        for (const Slice& x : sl) {
            if (!merged.empty() && merged.back().start == x.start && merged.back().end == x.end && merged.back().pad == x.pad)
                continue;
            if (!x.pad && !merged.empty() && !merged.back().pad && x.start <= merged.back().end + 32u)
                merged.back().end = std::max(merged.back().end, x.end);
            else
                merged.push_back(x);
        }
        // the x slices follow the stage in the slot (slot-relative offsets)
        uint32_t data_bytes = static_cast<uint32_t>((end - pos) * kItemBytes);
        for (size_t t = pos; t < end; ++t) data_bytes += static_cast<uint32_t>(its[t].bytes);
        uint32_t coef = data_bytes, copied = 0;  // slot bytes used / bytes the copies bring
        for (Slice& x : merged) {
            if (x.pad && (x.start & 1u)) {  // bulk copies start at an even element
                x.start -= 1;
            }
            x.off = coef;
            copied += r16((x.end - x.start) * 8ull * R);
            coef += r16((x.end - x.start) * 8ull * R) + (x.pad ? 16u : 0u);
        }
        if (coef > static_cast<uint32_t>(kSlotDataA) || merged.size() > static_cast<size_t>(kCopies)) return false;
        auto xoff = [&](const ALane& L) -> uint32_t {  // coef-area offset of x[xidx], in doubles
            const uint32_t pad = L.G > 1 ? 1u : 0u;
            for (const Slice& x : merged)
                if (x.pad == pad && x.start <= L.xidx && L.xidx + L.nf <= x.end) return x.off / 8 + (L.xidx - x.start) * static_cast<uint32_t>(R);
            throw std::logic_error("hmat: x slice");
        };
        // descriptors largest first (the rotating deal spreads the large ones over the warps)
        std::vector<size_t> ord;
        for (size_t t = pos; t < end; ++t) ord.push_back(t);
        std::stable_sort(ord.begin(), ord.end(), [&](size_t a2, size_t b2) { return its[a2].bytes > its[b2].bytes; });
        const size_t c0 = copies.size();
        copies.resize(c0 + kCopies, 0);
        for (size_t q = 0; q < merged.size(); ++q)
            copies[c0 + q] = copy_entry(merged[q].start, merged[q].off, r16((merged[q].end - merged[q].start) * 8ull * R), 0);
        while (arena.size() % 4) arena.push_back(0u);
        const uint64_t start = arena.size();
        arena.resize(start + ord.size() * (kItemBytes / 4), 0u);
        uint64_t cost = 0;
        for (size_t n = 0; n < ord.size(); ++n) {
            const AIt& t = its[ord[n]];
            AItem it{};
            it.word_off = static_cast<uint32_t>(arena.size() - start);
            it.nf = static_cast<uint16_t>(lanes[t.l0].nf);
            it.nl = static_cast<uint8_t>(t.nl);
            it.dest0 = lanes[t.l0].dest;
            it.rowbits = static_cast<uint16_t>(t.rowbits);
            it.gwords = static_cast<uint16_t>(t.gwords);
            it.final_ = static_cast<uint8_t>(lanes[t.l0].final_);
            const uint32_t G = lanes[t.l0].G, C = static_cast<uint32_t>(kALanes) / G;
            it.cshift = static_cast<uint8_t>(__builtin_ctz(G == 1 ? static_cast<uint32_t>(kALanes) : C));
            const size_t nrec = G == 1 ? t.nl : static_cast<size_t>(kALanes);
            it.nl = static_cast<uint8_t>(nrec);
            // physical lane l <- segment l % C, chunk l / C (G > 1): one 8-lane
            // shared-memory phase of the x loads reads two x chunks, not eight
            auto src_of = [&](size_t l) -> long {
                if (G == 1) return static_cast<long>(t.l0 + l);
                const size_t sg = l % C, g = l / C;
                return sg * G < t.nl ? static_cast<long>(t.l0 + sg * G + g) : -1L;
            };
            bool fast = it.nf % kARows == 0;
            std::vector<std::pair<uint64_t, uint32_t>> fast_rec;  // the records of a fast item (see a_item)
            const uint64_t rec0 = arena.size();
            arena.resize(rec0 + ((nrec + 3) & ~size_t(3)), 0u);
            const uint64_t data0 = arena.size();
            arena.resize(data0 + static_cast<uint64_t>(t.ngroups) * t.gwords, 0u);
            uint32_t P = 0;
            for (size_t q = 0; q < nrec; ++q) {
                const long li = src_of(q);
                if (li < 0) continue;  // idle lane: record 0
                const ALane& L = lanes[static_cast<size_t>(li)];
                const hcmx_descriptor& x = d.desc[L.buf];
                const unsigned w = x.bit_width, e = x.exp_bits, m = x.mant_bits;
                const unsigned fmt = x.scheme >= HCMX_RAW_F64 ? 3u + (x.scheme - HCMX_RAW_F64) : 0u;
                const uint32_t xo = xoff(L);
                if (xo >= 8192u || w > 64) throw std::logic_error("hmat: phase-A lane record");
                fast = fast && fmt == 0 && w <= 32 && e <= 10 && w == 1 + e + m && xo % 2 == 0;
                arena[rec0 + q] = w | (e << 7) | ((fmt ? 0u : m) << 11) | ((fmt ? fmt - 2u : 0u) << 17) | (xo << 19);
                fast_rec.push_back({rec0 + q, ((w - 1u) & 31u) | (e << 5) | (P << 9) | ((xo / 2u) << 19) | kARecValid});
                fast = fast && P < 1024u && xo / 2u < 4096u;
                lane_jobs.push_back({data0, L.buf, L.f0, L.nf, P, t.rowbits, t.gwords});
                if (keep_map)
                    h->segs[L.buf].push_back({data0, static_cast<uint32_t>(L.f0), L.nf, P,
                                              static_cast<uint16_t>(t.rowbits), static_cast<uint16_t>(t.gwords)});
                P += w;
            }
            it.body = fast ? 1 : 0;
            if (fast)
                for (const auto& fr : fast_rec) arena[fr.first] = fr.second;
            std::memcpy(arena.data() + start + n * (kItemBytes / 4), &it, kItemBytes);
            while (arena.size() % 4) arena.push_back(0u);
            cost += 60 + 40ull * t.ngroups * (fast ? 1 : 3);  // ~warp instructions
        }
        while (arena.size() % 4) arena.push_back(0u);
        Stage st{};
        st.item0 = static_cast<uint32_t>(a_items);
        st.byte_off = start * 4;
        st.bytes = static_cast<uint32_t>((arena.size() - start) * 4);
        st.nitems = static_cast<uint32_t>(ord.size());
        st.pad = cost;
        if (st.bytes != data_bytes) throw std::logic_error("hmat: phase-A stage size");
        st.coef_bytes = copied;  // what the copies complete on the barrier (expect_tx)
        check_copies(c0, copied);
        stages.push_back(st);
        a_items += ord.size();
        return true;
    }
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
        } else if (d.kind[l] == 2) {
            const int64_t k = d.rank[l];
            if (k < 0) throw invalid_argument("hmat: lowrank leaf indices");
            if (k > 0) {  // a rank-0 leaf has no buffers
                if (d.buf0[l] < 0 || d.buf0[l] + 2 > (int64_t)d.nbuffers)
                    throw invalid_argument("hmat: lowrank leaf indices");
                if (d.count[d.buf0[l]] != rows * k || d.count[d.buf0[l] + 1] != cols * k)
                    throw invalid_argument("hmat: lowrank factor size mismatch");
            }
        } else {
            throw invalid_argument("hmat: unsupported leaf kind (CodecDense, APLR / MP lowrank, CodecLowrank)");
        }
    }
    for (uint64_t b = 0; b < d.nbuffers; ++b) {
        const hcmx_descriptor& x = d.desc[b];
        if (x.scheme >= HCMX_RAW_F64) {  // uncompressed storage: 64 / 32 / 16-bit IEEE words
            static const unsigned rw[3] = {64, 32, 16};
            if (x.scheme > HCMX_RAW_F16 || x.bit_width != rw[x.scheme - HCMX_RAW_F64] || x.scale != 1.0)
                throw invalid_argument("hmat: invalid raw-storage descriptor");
        } else if (x.scheme > 3 || x.exp_bits < 2 || x.exp_bits > 11 || x.mant_bits < 2 || x.mant_bits > 52 ||
                   x.bit_width != bit_width(x.scheme, x.exp_bits, x.mant_bits)) {
            throw invalid_argument("hmat: invalid buffer descriptor");
        }
        if (d.poff[b] < 0 || d.plen[b] < 0 || (uint64_t)(d.poff[b] + d.plen[b]) > d.blob_bytes)
            throw corrupt_buffer("hmat: payload outside the blob");
        if ((uint64_t)d.plen[b] < payload_bytes(d.count[b], x.bit_width))
            throw corrupt_buffer("bitstream: payload ends inside a value");
    }
}

void build(const hcmx_hmat_desc& d, hcmx_hmat* h) {
    validate(d);
    Builder B(d, h);
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

    HostBlob hb;
    if (d.blob_on_device) {
        // a device-resident blob is read on the host through a lazily backed
        // mapping: only the byte ranges of this partition's buffers are copied
        // (and become resident), so one rank of a block-row partition does not
        // hold the whole matrix in host memory
        std::vector<std::pair<uint64_t, uint64_t>> rng;  // [begin, end)
        auto need = [&](int64_t b) {
            if (d.plen[b] > 0) rng.push_back({static_cast<uint64_t>(d.poff[b]), static_cast<uint64_t>(d.poff[b] + d.plen[b])});
        };
        for (uint64_t l : leaves) {
            const int64_t k = d.rank[l];
            const int64_t nb = d.kind[l] == 0 ? 1 : d.kind[l] == 1 ? 2 * k : (k > 0 ? 2 : 0);
            for (int64_t i = 0; i < nb; ++i) need(d.buf0[l] + i);
        }
        std::sort(rng.begin(), rng.end());
        hb.map(d.blob_bytes);
        uint64_t a = 0, e = 0;
        bool open = false;
        auto flush = [&]() {
            if (open) check_cuda(cudaMemcpy(hb.p + a, d.blob + a, e - a, cudaMemcpyDeviceToHost), "blob d2h");
        };
        for (const auto& r : rng) {
            if (open && r.first <= e + 65536) {
                e = std::max(e, r.second);
            } else {
                flush();
                a = r.first;
                e = r.second;
                open = true;
            }
        }
        flush();
        B.blob = hb.p;
        uint64_t need_bytes = 0;
        for (const auto& r : rng) need_bytes += r.second - r.first;
        B.arena.reserve(need_bytes / 4 + need_bytes / 40 + (1u << 20));  // + item / record overhead
    } else {
        B.blob = d.blob;
        B.arena.reserve(d.blob_bytes / 4 + d.blob_bytes / 40 + (1u << 20));
    }
    const bool stats = std::getenv("HCMX_BUILD_STATS") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto t_build = now();
    auto lap = [&](const char* what) {
        if (!stats) return;
        const auto t = now();
        std::fprintf(stderr, "[build] %s %.2f s\n", what, std::chrono::duration<double>(t - t_build).count());
        t_build = t;
    };
    lap("blob to host");

    uint64_t total_fields = 0;
    for (uint64_t b = 0; b < d.nbuffers; ++b) total_fields += d.count[b];
    B.keep_map = total_fields <= (1ull << 28);
    if (B.keep_map) h->segs.assign(d.nbuffers, {});

    // (buffer, first field) of rank column i of a lowrank leaf: one buffer per
    // column (APLR / MP, kind 1) or a slice of the U / V buffer (CodecLowrank, kind 2)
    auto wbuf = [&](uint64_t l, uint32_t i) -> std::pair<uint64_t, uint64_t> {
        if (d.kind[l] == 2) return {static_cast<uint64_t>(d.buf0[l]), static_cast<uint64_t>(i) * (d.row1[l] - d.row0[l])};
        return {static_cast<uint64_t>(d.buf0[l] + i), 0};
    };
    auto xbuf = [&](uint64_t l, uint32_t i) -> std::pair<uint64_t, uint64_t> {
        if (d.kind[l] == 2)
            return {static_cast<uint64_t>(d.buf0[l] + 1), static_cast<uint64_t>(i) * (d.col1[l] - d.col0[l])};
        return {static_cast<uint64_t>(d.buf0[l] + d.rank[l] + i), 0};
    };

    // per-leaf tables; rank-column ids (wcol / coef) and partial ranges are
    // assigned by the phase-A layout below, in the order its items' lanes take
    std::vector<int64_t> lr_id(d.nleaves, -1);
    std::vector<LeafA> leafa;
    std::vector<uint64_t> lr_leaf;  // leaf index of each lowrank leaf
    uint64_t npartial = 0;
    uint32_t ncols = 0;
    std::vector<RedCol> redcols;
    hcmx_memory_report& rep = h->report;
    rep = hcmx_memory_report{};
    for (uint64_t l : leaves) {
        const int64_t rows = d.row1[l] - d.row0[l], cols = d.col1[l] - d.col0[l];
        if (d.kind[l] == 0) {
            const hcmx_descriptor& x = d.desc[d.buf0[l]];
            const bool raw = x.scheme >= HCMX_RAW_F64;  // uncompressed FP64 leaf (StorageMode fp64 / MP)
            rep.dense_leaves++;
            if (raw) rep.dense_raw += d.plen[d.buf0[l]];
            else rep.dense_compressed += 20 + d.plen[d.buf0[l]];
            rep.uncompressed_equivalent += 8ull * rows * cols;
            rep.algorithmic_bytes += (raw ? 0 : 20) + payload_bytes(rows * cols, x.bit_width);
        } else {
            const uint32_t k = static_cast<uint32_t>(d.rank[l]);
            lr_id[l] = static_cast<int64_t>(leafa.size());
            LeafA L{};
            L.k = k;
            L.nchunks = static_cast<uint32_t>((cols + kAChunk - 1) / kAChunk);
            if (k >= (1u << 16) || L.nchunks >= (1u << 16)) throw invalid_argument("hmat: lowrank leaf too large");
            leafa.push_back(L);
            lr_leaf.push_back(l);
            const bool uniform = d.kind[l] == 2;  // CodecLowrank: one U and one V buffer, sigma = 1
            uint64_t bytes = uniform ? 4 : 8 + 8ull * k;  // APLRLowrank::byte_size (mixedprec.cpp:210-217)
            if (uniform && k > 0) {
                for (int f = 0; f < 2; ++f) {
                    const hcmx_descriptor& x = d.desc[d.buf0[l] + f];
                    const uint64_t n = f ? cols * k : rows * k;
                    const uint64_t hdr = x.scheme >= HCMX_RAW_F64 ? 0 : 20;
                    bytes += hdr + d.plen[d.buf0[l] + f];
                    rep.algorithmic_bytes += hdr + payload_bytes(n, x.bit_width);
                }
            }
            for (uint32_t i = 0; i < k && !uniform; ++i) {
                const hcmx_descriptor& xw = d.desc[wbuf(l, i).first];
                const hcmx_descriptor& xx = d.desc[xbuf(l, i).first];
                const uint64_t hdr = xw.scheme >= HCMX_RAW_F64 ? 0 : 20;
                bytes += 2 * hdr + d.plen[d.buf0[l] + i] + d.plen[d.buf0[l] + k + i];
                rep.algorithmic_bytes += 2 * hdr + payload_bytes(rows, xw.bit_width) + payload_bytes(cols, xx.bit_width);
            }
            if (!uniform) rep.algorithmic_bytes += 8ull * k;
            rep.lowrank_leaves++;
            rep.lowrank_compressed += bytes;
            rep.uncompressed_equivalent += 8ull * (rows + cols) * k;
        }
    }
    rep.algorithmic_bytes += 8ull * d.n_cols + 8ull * (h->re - h->rb);
    h->nlr = static_cast<uint32_t>(leafa.size());

    // ---- phase A: stripes of ~kAStripeBytes of X factors.  In a stripe, the
    // leaves that fit one chunk come first, grouped by width (so lanes of
    // several leaves fill an item and write consecutive wcol records), then the
    // chunked leaves, whose lanes run over (chunk, rank column) and write
    // consecutive partials.
    uint32_t nstripe_a = 0;
    std::vector<uint32_t> stripe_a = {0};
    {
        // stripe size: up to kAStripeBytes (32 stages: fewer partly filled last
        // stages and stripe claims; config 4 phase A -3 % against 8 stages),
        // smaller when the X factors of this handle would give fewer than ~6
        // stripes per CTA slot (2 per SM) -- else the slowest stripe sets the
        // phase time (config 3, 1.1 GB: 8 stages per stripe measured best, 12 or
        // more +3.5 %)
        uint64_t xbytes_all = 0;
        for (uint64_t l : leaves)
            if (d.kind[l] != 0)
                for (uint32_t i = 0; i < leafa[lr_id[l]].k; ++i)
                    xbytes_all += B.words_of(xbuf(l, i).first, d.col1[l] - d.col0[l]) * 4;
        const uint64_t stripe_target =
            std::max<uint64_t>(2ull * kStageBytesA, std::min<uint64_t>(kAStripeBytes, xbytes_all / (19ull * kCtasA * 148 / 3)));
        std::vector<uint32_t> pend;  // lowrank ids of the current stripe
        uint64_t stripe_bytes = 0;
        std::vector<ALane> lanes;
        auto flush = [&]() {
            if (pend.empty()) return;
            lanes.clear();
            std::vector<uint32_t> single, chunked;
            for (uint32_t id : pend) (leafa[id].nchunks == 1 ? single : chunked).push_back(id);
            auto cols_of = [&](uint32_t id) { return d.col1[lr_leaf[id]] - d.col0[lr_leaf[id]]; };
            std::stable_sort(single.begin(), single.end(), [&](uint32_t a2, uint32_t b2) { return cols_of(a2) < cols_of(b2); });
            for (uint32_t id : single) {
                LeafA& L = leafa[id];
                const uint64_t l = lr_leaf[id];
                L.colbase = ncols;
                ncols += L.k;
                for (uint32_t i = 0; i < L.k; ++i) {
                    const auto xb = xbuf(l, i);
                    lanes.push_back({xb.first, xb.second, static_cast<uint32_t>(cols_of(id)),
                                     static_cast<uint32_t>(d.col0[l]), L.colbase + i, 1, 1, 0});
                }
            }
            for (uint32_t id : chunked) {
                // whole 64-row chunks in groups of G (a power of two <= kAGroupMax
                // dividing their count) summed in-warp; a ragged last chunk is a
                // group of its own.  One group: the result is final.
                LeafA& L = leafa[id];
                const uint64_t l = lr_leaf[id];
                const uint64_t cols = static_cast<uint64_t>(cols_of(id));
                const uint32_t nfull = static_cast<uint32_t>(cols / kAChunk), rag = static_cast<uint32_t>(cols % kAChunk);
                uint32_t G = 1;
                // R right-hand sides stage R x slices per chunk: smaller segments
                // keep a segment's x (G chunks x 64 rows x R doubles) a fraction of a slot
                const uint32_t gmax = h->R == 1 ? static_cast<uint32_t>(kAGroupMax) : (h->R == kMultiR ? kAGroupMaxMulti : 1u);
                while (2 * G <= gmax && nfull % (2 * G) == 0) G *= 2;
                const uint32_t ngrp = nfull / G + (rag ? 1u : 0u);
                L.colbase = ncols;
                ncols += L.k;
                L.nchunks = ngrp;
                const uint32_t fin = ngrp == 1 ? 1u : 0u;
                if (!fin) {
                    L.pbase = static_cast<uint32_t>(npartial);
                    for (uint32_t i = 0; i < L.k; ++i) redcols.push_back({L.colbase + i, L.pbase + i, L.k, ngrp});
                    npartial += static_cast<uint64_t>(ngrp) * L.k;
                }
                for (uint32_t grp = 0; grp < ngrp; ++grp) {
                    const bool ragged = grp * G >= nfull;
                    const uint32_t gs = ragged ? 1u : G;
                    for (uint32_t i = 0; i < L.k; ++i) {
                        const auto xb = xbuf(l, i);
                        const uint32_t dest = fin ? L.colbase + i : L.pbase + grp * L.k + i;
                        for (uint32_t g = 0; g < gs; ++g) {
                            const uint64_t f0 = static_cast<uint64_t>(ragged ? nfull : grp * G + g) * kAChunk;
                            const uint32_t nf = ragged ? rag : static_cast<uint32_t>(kAChunk);
                            lanes.push_back({xb.first, xb.second + f0, nf, static_cast<uint32_t>(d.col0[l] + f0), dest,
                                             fin, gs, g});
                        }
                    }
                }
            }
            if (npartial >= (1ull << 32) || ncols >= (1u << 31)) throw invalid_argument("hmat: too many rank columns");
            // one stripe is one CTA's serial work: a leaf whose X factor is larger
            // than the stripe target (the top-level blocks: 8192 ... 32768
            // columns) is cut at segment boundaries into several stripes, so its
            // columns are decoded by several CTAs (segments write separate
            // partials, k_reduce adds them in fixed order)
            std::vector<ALane> part;
            uint64_t pbytes = 0;
            for (size_t i = 0; i < lanes.size(); ++i) {
                const ALane& L = lanes[i];
                if (L.g == 0 && pbytes >= stripe_target && !part.empty()) {
                    B.emit_stripe_a(part);
                    stripe_a.push_back(static_cast<uint32_t>(B.stages.size()));
                    ++nstripe_a;
                    part.clear();
                    pbytes = 0;
                }
                part.push_back(L);
                pbytes += (static_cast<uint64_t>(L.nf) * B.width(L.buf) + 7) / 8;
            }
            if (!part.empty()) {
                B.emit_stripe_a(part);
                stripe_a.push_back(static_cast<uint32_t>(B.stages.size()));
                ++nstripe_a;
            }
            pend.clear();
            stripe_bytes = 0;
        };
        // Leaves in column-cluster order: the admissible blocks of one column
        // cluster share their x slice, so an item's lanes (rank columns of
        // consecutive leaves) and a stage's items mostly read ONE staged slice --
        // fewer coefficient copies per stage and fewer slot bytes spent on x
        // (in leaf order a third of a stage's packed bytes).
        std::vector<uint64_t> leaves_a;
        for (uint64_t l : leaves)
            if (d.kind[l] != 0) leaves_a.push_back(l);
#if HCMX_A_SIGMA
        std::stable_sort(leaves_a.begin(), leaves_a.end(), [&](uint64_t a2, uint64_t b2) {
            if (d.col0[a2] != d.col0[b2]) return d.col0[a2] < d.col0[b2];
            return d.col1[a2] < d.col1[b2];
        });
#endif
        for (uint64_t l : leaves_a) {
            const uint32_t id = static_cast<uint32_t>(lr_id[l]);
            pend.push_back(id);
            for (uint32_t i = 0; i < leafa[id].k; ++i)
                stripe_bytes += B.words_of(xbuf(l, i).first, d.col1[l] - d.col0[l]) * 4;
            if (stripe_bytes >= stripe_target) flush();
        }
        flush();
    }
    // rank-column tables in the order phase A assigned
    const uint32_t rb = rec_bytes_rt(h->R);
    std::vector<uint8_t> wrec(static_cast<size_t>(ncols + 4) * rb, 0);  // + 4: bulk copies may round up
    std::vector<double> coef(ncols + 4, 0.0);
    for (uint32_t id = 0; id < leafa.size(); ++id) {
        const uint64_t l = lr_leaf[id];
        const bool uniform = d.kind[l] == 2;
        for (uint32_t i = 0; i < leafa[id].k; ++i) {
            const hcmx_descriptor& xw = d.desc[wbuf(l, i).first];
            const hcmx_descriptor& xx = d.desc[xbuf(l, i).first];
            const ColPar cp = col_par(xw);
            // record {c[R] (phase A writes it), mask, mul, packed, w}
            const uint32_t par[4] = {cp.mask, cp.mul, cp.packed, xw.bit_width};
            std::memcpy(wrec.data() + static_cast<size_t>(leafa[id].colbase + i) * rb + 8 * h->R, par, sizeof(par));
            // complex arenas: phase A leaves alpha scale_X (X^T x); k_ccombine applies
            // sigma and the W scales while pairing the real / imaginary halves
            coef[leafa[id].colbase + i] = h->cplx ? xx.scale : (uniform ? 1.0 : d.sigma[d.sig0[l] + i]) * xx.scale * xw.scale;
        }
    }
    std::vector<CPair> pairs;  // complex: rank pairs (Ur_j | Vr_j, Ui_j | Vi_j) of every lowrank leaf
    if (h->cplx) {
        for (uint32_t id = 0; id < leafa.size(); ++id) {
            const uint64_t l = lr_leaf[id];
            const uint32_t k2 = leafa[id].k, k = k2 / 2;
            if (k2 % 2) throw invalid_argument("hmat: complex lowrank leaf with odd real rank");
            for (uint32_t j = 0; j < k; ++j)
                pairs.push_back({leafa[id].colbase + j, leafa[id].colbase + k + j, d.sigma[d.sig0[l] + j],
                                 d.desc[wbuf(l, j).first].scale, d.desc[wbuf(l, k + j).first].scale});
        }
    }
    rep.stages_a = B.stages.size();
    lap("phase-A layout");

    // ---- phase B: one stripe per block of kR rows
    const uint64_t nblocks = (h->re - h->rb + kR - 1) / kR;
    std::vector<std::vector<uint32_t>> block_leaves(nblocks);
    for (uint64_t l : leaves) {
        const uint64_t a = std::max<uint64_t>(d.row0[l], h->rb) - h->rb;
        const uint64_t b = std::min<uint64_t>(d.row1[l], h->re) - h->rb;
        for (uint64_t blk = a / kR; blk * kR < b; ++blk) block_leaves[blk].push_back(static_cast<uint32_t>(l));
    }
    // dense leaves first in every row block: their stages need nothing from
    // phase A, so a phase-B CTA that starts while phase A drains (programmatic
    // dependent launch) has work before it must wait for the coefficients
    for (auto& bl : block_leaves)
        std::stable_partition(bl.begin(), bl.end(), [&](uint32_t l) { return d.kind[l] == 0; });
    const size_t b_ws0 = B.stages.size();
    std::vector<uint32_t> stripe_b = {static_cast<uint32_t>(B.stages.size())};
    {
        std::vector<Spec<BItem>> specs;
        uint64_t unit = 0;
        for (uint64_t blk = 0; blk < nblocks; ++blk) {
            specs.clear();
            const uint64_t b0 = h->rb + blk * kR, b1 = std::min<uint64_t>(b0 + kR, h->re);
            for (uint32_t l : block_leaves[blk]) {
                ++unit;  // one item key per (leaf, row block)
                const int64_t rows = d.row1[l] - d.row0[l], cols = d.col1[l] - d.col0[l];
                const uint64_t r0 = std::max<uint64_t>(d.row0[l], b0), r1 = std::min<uint64_t>(d.row1[l], b1);
                const uint64_t nr = r1 - r0, roff = r0 - d.row0[l];
                if (d.kind[l] == 0) {
                    const uint64_t b = d.buf0[l];
                    const auto groups = column_groups(static_cast<uint32_t>(cols), 1,
                                                      [&](uint32_t) { return B.words_of(b, nr); });
                    for (const auto& gr : groups) {
                        const int64_t c0 = gr.first;
                        const uint32_t nc = gr.second;
                        Spec<BItem> sp{};
                        sp.seg0 = static_cast<uint32_t>(B.segs.size());
                        sp.nseg = nc;
                        for (uint32_t c = 0; c < nc; ++c) {
                            B.segs.push_back({b, static_cast<uint64_t>((c0 + c) * rows + roff), nr});
                            sp.words += B.words_of(b, nr);
                        }
                        BItem& it = sp.it;
                        it.src = static_cast<uint32_t>(d.col0[l] + c0);
                        it.nseg = static_cast<uint8_t>(nc);
                        it.kind = 0;
                        it.ra = static_cast<uint8_t>(r0 - b0);
                        it.nr = static_cast<uint8_t>(nr);
                        it.dpacked = col_par(d.desc[b]).packed;
                        it.mode = static_cast<uint8_t>(it.dpacked >> 24);
                        it.fcase = bcase_of(r0 - b0, nr, it.mode);
                        it.scale = d.desc[b].scale;
                        sp.elem = it.src;
                        // x slice of the dense leaf's columns; the imaginary part of a
                        // complex dense block reads the swapped x (-Im x, Re x)
                        sp.sl_table = (h->cplx && d.dense_imag && d.dense_imag[l]) ? 2 : 0;
                        sp.sl_start = static_cast<uint32_t>(d.col0[l]);
                        sp.sl_count = static_cast<uint32_t>(cols);
                        sp.cost = 3 * nr + 128;  // ~decode instructions (x8) of one column segment
                        sp.unit = unit * 8 + it.mode;
                        specs.push_back(sp);
                    }
                } else {
                    const LeafA& L = leafa[lr_id[l]];
                    const auto groups = column_groups(L.k, 1, [&](uint32_t i) { return B.words_of(wbuf(l, i).first, nr); });
                    for (const auto& gr : groups) {
                        const uint32_t g = gr.first, ng = gr.second;
                        Spec<BItem> sp{};
                        sp.seg0 = static_cast<uint32_t>(B.segs.size());
                        sp.nseg = ng;
                        for (uint32_t i = g; i < g + ng; ++i) {
                            const auto wb2 = wbuf(l, i);
                            B.segs.push_back({wb2.first, wb2.second + roff, nr});
                            sp.words += B.words_of(wb2.first, nr);
                        }
                        BItem& it = sp.it;
                        it.nseg = static_cast<uint8_t>(ng);
                        it.kind = 1;
                        it.ra = static_cast<uint8_t>(r0 - b0);
                        it.nr = static_cast<uint8_t>(nr);
                        it.src = L.colbase + g;
                        it.mode = static_cast<uint8_t>(col_par(d.desc[wbuf(l, g).first]).packed >> 24);
                        it.fcase = bcase_of(r0 - b0, nr, it.mode);
                        sp.elem = it.src;
                        sp.sl_table = 1;  // phase-A results of the leaf
                        sp.sl_start = L.colbase;
                        sp.sl_count = L.k;
                        sp.cost = 3 * nr + 128;
                        sp.unit = unit * 8 + it.mode;  // items never mix decode modes
                        specs.push_back(sp);
                    }
                }
            }
            if (h->R == 1) B.emit_stripe<BItem, kBLRGroup, kNWB>(specs, B.bitems);
            else if (h->R == kMultiR) B.emit_stripe<BItem, kBLRGroup, nwb<kMultiR>()>(specs, B.bitems);
            else B.emit_stripe<BItem, kBLRGroup, nwb<kMultiR2>()>(specs, B.bitems);
            stripe_b.push_back(static_cast<uint32_t>(B.stages.size()));
        }
    }
    rep.stages_b = B.stages.size() - b_ws0;
    lap("phase-B layout");
    if (std::getenv("HCMX_BUILD_STATS")) {  // profiling aid: copies / items / bytes per stage
        for (int ph = 0; ph < 2; ++ph) {
            const size_t s0 = ph ? b_ws0 : 0, s1 = ph ? B.stages.size() : b_ws0;
            uint64_t nc = 0, cb = 0, db = 0, ni = 0;
            for (size_t st = s0; st < s1; ++st) {
                for (size_t q = 0; q < kCopies; ++q) nc += B.copies[st * kCopies + q] >> 63;
                cb += B.stages[st].coef_bytes;
                db += B.stages[st].bytes;
                ni += B.stages[st].nitems;
            }
            const double n = std::max<double>(1.0, double(s1 - s0));
            std::fprintf(stderr, "[build %c] stages %zu: per stage %.1f copies, %.1f items, %.0f data B, %.0f coef B\n",
                         ph ? 'B' : 'A', s1 - s0, nc / n, ni / n, db / n, cb / n);
        }
    }
    B.segs.clear();
    B.segs.shrink_to_fit();
    B.place_all();
    lap("bit placement");
    while (B.arena.size() % 4) B.arena.push_back(0u);
    B.arena.resize(B.arena.size() + 8, 0u);  // tail slack
    if (B.stages.size() >= (1ull << 31)) throw invalid_argument("hmat: too many stages");

    // ---- upload
    cudaStream_t s = h->stream;
    auto up = [&](DevBuf& dst, const void* src, size_t bytes) {
        dst.alloc(std::max<size_t>(bytes, 16));
        if (bytes) h2d(dst.p, src, bytes, s);
    };
    up(h->arena, B.arena.data(), B.arena.size() * 4);
    up(h->stages, B.stages.data(), B.stages.size() * sizeof(Stage));
    up(h->copies, B.copies.data(), B.copies.size() * sizeof(uint64_t));
    h->work.alloc(16);
    check_cuda(cudaMemsetAsync(h->work.p, 0, 16, s), "memset");
    // stripes in decreasing estimated cost: the persistent CTAs claim the big ones
    // first, so they finish together (every stripe's result is independent of
    // which CTA computes it, so the order is free)
    auto lpt = [&](const std::vector<uint32_t>& range, bool with_block) {
        std::vector<std::array<uint32_t, 4>> v;
        std::vector<uint64_t> cost;
        for (size_t i = 0; i + 1 < range.size(); ++i) {
            uint64_t c = 0;
            for (uint32_t s2 = range[i]; s2 < range[i + 1]; ++s2) c += B.stages[s2].pad;
            v.push_back({range[i], range[i + 1], with_block ? static_cast<uint32_t>(i) : 0u, 0u});
            cost.push_back(c);
        }
        std::vector<size_t> ord(v.size());
        for (size_t i = 0; i < ord.size(); ++i) ord[i] = i;
        std::stable_sort(ord.begin(), ord.end(), [&](size_t a, size_t b) { return cost[a] > cost[b]; });
        std::vector<std::array<uint32_t, 4>> out;
        for (size_t i : ord) out.push_back(v[i]);
        return out;
    };
    const auto sa = lpt(stripe_a, false);
    // phase-B stripes: one row block each.  With too few blocks to keep every CTA
    // slot busy (one rank of a block-row partition), a block is cut into up to
    // kMaxPieces stage ranges of similar cost; their partial row sums go to
    // ypart and k_combine adds them (fixed order, beta y once).
    const uint64_t nb_rows = stripe_b.size() - 1;
    const uint64_t want = static_cast<uint64_t>(kCtasB) * 148;  // one stripe per CTA slot
    const char* mp_env = std::getenv("HCMX_MAX_PIECES");  // test / profiling knob (1: never split)
    const uint64_t max_pieces = mp_env ? std::max(1, std::min(std::atoi(mp_env), static_cast<int>(kMaxPieces)))
                                       : kMaxPieces;
    // (measured on config 3 row partitions: 128 blocks split 3 ways 85 -> 71 us,
    // 256 blocks split 2 ways 100 -> 109 us: only blocks fewer than the SMs split)
    const uint32_t S = 2 * nb_rows > want ? 1u
                                          : static_cast<uint32_t>(std::min<uint64_t>(max_pieces, (want + nb_rows - 1) / nb_rows));
    std::vector<std::array<uint32_t, 4>> bv;
    std::vector<uint64_t> bcost;
    std::vector<uint8_t> dense_only;  // HCMX_COSCHED: stripes that never wait for phase A
    std::vector<uint8_t> npieces(std::max<uint64_t>(nb_rows, 1), 0);
    // HCMX_COSCHED (experiment, off): every row block with dense and lowrank
    // stages is cut into two pieces at its first stage that reads phase-A
    // results, and the dense pieces are claimed first -- phase B's CTAs work on
    // them while phase A still runs on the same SMs (phase A at one CTA per SM
    // leaves room for one of B's).  Measured slower: config 4 4.45 vs 3.89 ms
    // (phase A at one CTA per SM loses more than the overlap gains), 3.88 ms
    // with phase A at two CTAs per SM (no co-residence, dense pieces first).
    auto needs_a = [&](uint32_t st) {
        for (size_t q = static_cast<size_t>(st) * kCopies; q < static_cast<size_t>(st + 1) * kCopies; ++q)
            if ((B.copies[q] >> 63) && ((B.copies[q] >> 60) & 3u) == 1u) return true;
        return false;
    };
    for (uint64_t i = 0; i < nb_rows; ++i) {
        const uint32_t s0 = stripe_b[i], s1 = stripe_b[i + 1];
        if (HCMX_COSCHED && S == 1) {
            uint32_t sx = s0;
            while (sx < s1 && !needs_a(sx)) ++sx;
            uint64_t c1 = 0, c2 = 0;
            for (uint32_t s2 = s0; s2 < sx; ++s2) c1 += B.stages[s2].pad;
            for (uint32_t s2 = sx; s2 < s1; ++s2) c2 += B.stages[s2].pad;
            if (sx == s0 || sx == s1) {  // dense only or lowrank only: one piece
                bv.push_back({s0, s1, static_cast<uint32_t>(i), 0u});
                bcost.push_back(sx == s1 ? c1 : c2);
                dense_only.push_back(sx == s1 ? 1u : 0u);
            } else {
                npieces[i] = 2;
                bv.push_back({s0, sx, static_cast<uint32_t>(i), 1u});
                bcost.push_back(c1);
                dense_only.push_back(1u);
                bv.push_back({sx, s1, static_cast<uint32_t>(i), 2u});
                bcost.push_back(c2);
                dense_only.push_back(0u);
            }
            continue;
        }
        const uint32_t P = std::min<uint32_t>(S, s1 - s0);
        uint64_t total = 0;
        for (uint32_t s2 = s0; s2 < s1; ++s2) total += B.stages[s2].pad;
        if (P <= 1) {
            bv.push_back({s0, s1, static_cast<uint32_t>(i), 0u});
            bcost.push_back(total);
            continue;
        }
        npieces[i] = static_cast<uint8_t>(P);
        uint32_t a = s0;
        uint64_t acc = 0;
        for (uint32_t q = 0; q < P; ++q) {  // contiguous pieces, cut at cumulative cost q / P
            uint32_t b = a;
            uint64_t c = 0;
            const uint64_t target = total * (q + 1) / P;
            while (b < s1 && (q + 1 == P || (b == a || acc + c + B.stages[b].pad / 2 <= target)) &&
                   s1 - b > P - 1 - q) {
                c += B.stages[b].pad;
                ++b;
            }
            if (q + 1 == P) {
                while (b < s1) c += B.stages[b++].pad;
            }
            bv.push_back({a, b, static_cast<uint32_t>(i), q + 1});
            bcost.push_back(c);
            acc += c;
            a = b;
        }
    }
    std::vector<size_t> bord(bv.size());
    for (size_t i = 0; i < bord.size(); ++i) bord[i] = i;
    std::stable_sort(bord.begin(), bord.end(), [&](size_t a2, size_t b2) {
        if (!dense_only.empty() && dense_only[a2] != dense_only[b2]) return dense_only[a2] > dense_only[b2];
        return bcost[a2] > bcost[b2];
    });
    std::vector<std::array<uint32_t, 4>> sb;
    for (size_t i : bord) sb.push_back(bv[i]);
    uint32_t SP = S;
    if (HCMX_COSCHED && S == 1)
        for (uint8_t q : npieces) SP = std::max<uint32_t>(SP, q);
    h->pieces = SP > 1 ? SP : 0;
    if (SP > 1) {
        up(h->npieces, npieces.data(), npieces.size());
        h->ypart.alloc(static_cast<size_t>(SP) * (h->re - h->rb) * h->R * 8);
    }
    up(h->stripe_a, sa.data(), sa.size() * 16);
    up(h->stripe_b, sb.data(), sb.size() * 16);
    up(h->wcol, wrec.data(), wrec.size());
    up(h->coef, coef.data(), coef.size() * 8);
    if (h->cplx) {
        h->ncpairs = static_cast<uint32_t>(pairs.size());
        up(h->cpairs, pairs.data(), pairs.size() * sizeof(CPair));
        h->xswap.alloc((d.n_cols + 4) * h->R * 8);
        check_cuda(cudaMemsetAsync(h->xswap.p, 0, h->xswap.bytes, s), "memset");
    }
    h->xpad.alloc((d.n_cols + 4) * 8);
    check_cuda(cudaMemsetAsync(h->xpad.p, 0, h->xpad.bytes, s), "memset");
    h->partial.alloc(std::max<size_t>(16, npartial * 8 * h->R));
    // columns with >= kRedLong chunks first (one warp each in k_reduce)
    std::stable_partition(redcols.begin(), redcols.end(), [](const RedCol& r) { return r.nchunks >= kRedLong; });
    h->nred_long = static_cast<uint32_t>(
        std::count_if(redcols.begin(), redcols.end(), [](const RedCol& r) { return r.nchunks >= kRedLong; }));
    up(h->redcols, redcols.data(), redcols.size() * sizeof(RedCol));
    h->nred = static_cast<uint32_t>(redcols.size());
    stream_sync(s);
    h->nstripe_a = nstripe_a;
    h->nblocks = static_cast<uint32_t>(sb.size());  // phase-B stripes
    lap("upload");
    rep.device_arena_bytes = B.arena.size() * 4;
    rep.device_table_bytes = B.stages.size() * (sizeof(Stage) + kCopies * 8) + B.bitems.size() * sizeof(BItem) +
                             B.a_items * sizeof(AItem) +
                             wrec.size() + coef.size() * 8;
    rep.overhead = rep.device_table_bytes;
}

Params make_params(hcmx_hmat* h, double alpha, double beta, double* y) {
    Params p{};
    p.arena = h->arena.as<uint8_t>();
    p.stages = h->stages.as<Stage>();
    p.stripe_a = h->stripe_a.as<uint4>();
    p.stripe_b = h->stripe_b.as<uint4>();
    p.copies = h->copies.as<uint64_t>();
    p.work = h->work.as<unsigned>();
    p.nstripe_a = h->nstripe_a;
    p.nblocks = h->nblocks;
    p.coef = h->coef.as<double>();
    p.wrec = h->wcol.as<uint8_t>();
    p.partial = h->partial.as<double>();
    p.ypart = h->ypart.as<double>();
    p.x = h->xpad.as<double>();  // padded, 16-byte aligned copy of x (bulk copies)
    p.y = y;
    p.row_begin = static_cast<uint32_t>(h->rb);
    p.row_end = static_cast<uint32_t>(h->re);
    p.alpha = alpha;
    p.beta = beta;
    p.bias = 1023ull << 52;
    return p;
}

// dx, dy: n-vectors (h->R == 1) or n x R row-major blocks (h->R == kMultiR)
void run_matvec(hcmx_hmat* h, double alpha, const double* dx, double beta, double* dy, cudaStream_t s) {
    // per-device setup (kernel attributes are per device; one process may drive several)
    struct DevInfo {
        bool ready = false;
        int nsm = 148;
    };
    static std::mutex dev_mu;
    static DevInfo dev_info[64];
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    if (dev < 0 || dev >= 64) throw invalid_argument("matvec: device ordinal out of range");
    int nsm;
    {
        std::lock_guard<std::mutex> g(dev_mu);
        DevInfo& di = dev_info[dev];
        if (!di.ready) {
            const int sm = static_cast<int>(kSmemBytes), sma = static_cast<int>(kSmemBytesA);
            check_cuda(cudaFuncSetAttribute(k_phase_a<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sma), "smem attr");
            check_cuda(cudaFuncSetAttribute(k_phase_b<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm), "smem attr");
            check_cuda(cudaFuncSetAttribute(k_phase_a<kMultiR>, cudaFuncAttributeMaxDynamicSharedMemorySize, sma),
                       "smem attr");
            check_cuda(cudaFuncSetAttribute(k_phase_b<kMultiR>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm),
                       "smem attr");
            check_cuda(cudaFuncSetAttribute(k_phase_a<kMultiR2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sma),
                       "smem attr");
            check_cuda(cudaFuncSetAttribute(k_phase_b<kMultiR2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm),
                       "smem attr");
            check_cuda(cudaDeviceGetAttribute(&di.nsm, cudaDevAttrMultiProcessorCount, dev), "SM count");
            di.ready = true;
        }
        nsm = di.nsm;
    }
    const int R = h->R;
    std::lock_guard<std::mutex> hold(h->mu);
    if (!h->last) check_cuda(cudaEventCreateWithFlags(&h->last, cudaEventDisableTiming), "event");
    else if (h->last_stream != s) check_cuda(cudaStreamWaitEvent(s, h->last, 0), "stream wait");
    struct Mark {  // record the product's end on every exit path
        hcmx_hmat* h;
        cudaStream_t s;
        ~Mark() {
            cudaEventRecord(h->last, s);
            h->last_stream = s;
        }
    } mark{h, s};
    h->last_launches = 0;
    if (alpha == 0.0) {  // y = beta y without touching M
        const uint64_t n = (h->re - h->rb) * R;
        k_scale<<<(int)std::min<uint64_t>((n + 255) / 256, 4096), 256, 0, s>>>(dy + h->rb * R, n, beta);
        check_cuda(cudaGetLastError(), "scale launch");
        h->last_launches = 1;
        return;
    }
    // x slices are bulk-copied from an even index in 16-byte units: read x in
    // place when that stays inside it (16-byte aligned, even length), else from
    // the padded copy (R > 1: the caller's n x R block, allocated aligned)
    const bool direct = R > 1 || dx == h->xpad.as<double>() ||
                        (reinterpret_cast<uintptr_t>(dx) % 16 == 0 && h->n_cols % 2 == 0);
    if (!direct) check_cuda(cudaMemcpyAsync(h->xpad.p, dx, h->n_cols * 8, cudaMemcpyDeviceToDevice, s), "x copy");
    Params p = make_params(h, alpha, beta, dy);
    if (direct) p.x = dx;
    if (h->cplx) {  // the swapped right-hand sides of the imaginary dense parts
        p.x2 = h->xswap.as<double>();
        const uint64_t npairs = h->n_cols * R / 2;
        k_xswap<<<static_cast<int>(std::min<uint64_t>((npairs + 255) / 256, 4ull * nsm)), 256, 0, s>>>(
            dx, h->xswap.as<double>(), npairs);
        check_cuda(cudaGetLastError(), "xswap launch");
        h->last_launches++;
    }
    static const int debug_knob = [] {
        const char* e = std::getenv("HCMX_DEBUG");
        return e ? std::atoi(e) : 0;
    }();
    p.debug = debug_knob;
    hcmx_hmat::Rec rec{};
    if (h->timing) {
        rec = {take_event(h), take_event(h), take_event(h)};
        check_cuda(cudaEventRecord(rec.a0, s), "event");
    }
    // the stripe counters: phase A resets B's and B resets A's for the next
    // product (both start at zero); a product without phase A resets here
    const bool run_a = h->nlr && h->nstripe_a;
    if (!run_a) check_cuda(cudaMemsetAsync(h->work.p, 0, 8, s), "work counters");
    cudaLaunchAttribute pdl[1];
    pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl[0].val.programmaticStreamSerializationAllowed = 1;
    auto launch = [&](auto kernel, uint32_t grid, int threads, size_t smem, bool after_kernel, auto... args) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(threads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cfg.attrs = pdl;
        cfg.numAttrs = after_kernel && !h->timing ? 1 : 0;  // events between kernels: plain launches
        check_cuda(cudaLaunchKernelEx(&cfg, kernel, args...), "matvec launch");
        h->last_launches++;
    };
    const uint32_t ga = std::min<uint32_t>(h->nstripe_a, kCtasA * nsm), gb = std::min<uint32_t>(h->nblocks, kCtasB * nsm);
    const uint32_t gr = (h->nred_long + 7) / 8 + (h->nred - h->nred_long + 255) / 256;
    const RedCol* rc = h->redcols.as<RedCol>();
    const uint32_t gc = static_cast<uint32_t>(std::min<uint64_t>(((h->re - h->rb) * R + 255) / 256, 4 * nsm));
    auto chain = [&](auto rt) {
        constexpr int RR = decltype(rt)::value;
        if (run_a) launch(k_phase_a<RR>, ga, kThreadsA, kSmemBytesA, false, p);
        if (h->nred) launch(k_reduce<RR>, gr, 256, 0, true, p, rc, h->nred_long, h->nred);
        if (RR > 1 && h->cplx && h->ncpairs)
            launch(k_ccombine<RR>, std::min<uint32_t>((h->ncpairs + 255) / 256, 8 * nsm), 256, 0, true, p,
                   h->cpairs.as<CPair>(), h->ncpairs);
        if (h->timing) check_cuda(cudaEventRecord(rec.a1, s), "event");
        if (h->nblocks) launch(k_phase_b<RR>, gb, (nwb<RR>() + kNProd) * 32, kSmemBytes, run_a, p);
        if (h->pieces) launch(k_combine<RR>, gc, 256, 0, true, p, h->npieces.as<uint8_t>());
    };
    if (R == 1) chain(std::integral_constant<int, 1>{});
    else if (R == kMultiR) chain(std::integral_constant<int, kMultiR>{});
    else chain(std::integral_constant<int, kMultiR2>{});
    check_cuda(cudaGetLastError(), "matvec launch");
#ifdef HCMX_PROF
    static const bool prof_env = std::getenv("HCMX_PROF") != nullptr;
    if (prof_env) {
        unsigned long long v[2][8], ts[2][4];
        check_cuda(cudaStreamSynchronize(s), "prof sync");
        check_cuda(cudaMemcpyFromSymbol(v, g_prof, sizeof(v)), "prof read");
        check_cuda(cudaMemcpyFromSymbol(ts, g_ts, sizeof(ts)), "prof read");
        const unsigned long long z[2][8] = {};
        check_cuda(cudaMemcpyToSymbol(g_prof, z, sizeof(z)), "prof reset");
        const unsigned long long zt[2][4] = {{~0ull, 0, 0, 0}, {~0ull, 0, 0, 0}};
        check_cuda(cudaMemcpyToSymbol(g_ts, zt, sizeof(zt)), "prof reset");
        for (int ph = 0; ph < 2; ++ph) {
            const double w = v[ph][4] ? double(v[ph][4]) : 1.0, c = v[ph][7] ? double(v[ph][7]) : 1.0;
            std::fprintf(stderr,
                         "[prof %c] per consumer warp: wait_full %.1f us busy %.1f us stripe_end %.1f us | per producer: "
                         "wait_empty %.1f us total %.1f us (1.965 GHz)\n",
                         ph ? 'B' : 'A', v[ph][0] / w / 1965.0, v[ph][1] / w / 1965.0, v[ph][5] / w / 1965.0,
                         v[ph][2] / c / 1965.0, v[ph][3] / c / 1965.0);
            if (ts[ph][0] != ~0ull)
                std::fprintf(stderr, "[prof %c] CTA start: avg +%.1f us; CTA end: avg +%.1f us, last +%.1f us\n",
                             ph ? 'B' : 'A', (ts[ph][3] / c * 256.0 - ts[ph][0]) / 1e3, (ts[ph][2] / c * 256.0 - ts[ph][0]) / 1e3,
                             (ts[ph][1] - ts[ph][0]) / 1e3);
        }
    }
#endif
    if (h->timing) {
        check_cuda(cudaEventRecord(rec.b1, s), "event");
        h->pending.push_back(rec);
        h->calls++;
        if (h->pending.size() > 1024) drain_timing(h);
    }
}

// w-bit field at bit `pos` of a byte stream padded by >= 16 readable bytes
inline uint64_t get_field(const uint8_t* src, uint64_t pos, unsigned w) {
    uint64_t lo, hi;
    std::memcpy(&lo, src + (pos >> 3), 8);
    std::memcpy(&hi, src + (pos >> 3) + 8, 8);
    const unsigned sh = pos & 7u;
    uint64_t v = sh ? (lo >> sh) | (hi << (64 - sh)) : lo;
    return w == 64 ? v : v & ((1ull << w) - 1);
}
inline void put_field(uint8_t* dst, uint64_t pos, unsigned w, uint64_t v) {  // dst zeroed, padded
    const unsigned sh = pos & 7u;
    uint64_t lo, hi;
    std::memcpy(&lo, dst + (pos >> 3), 8);
    std::memcpy(&hi, dst + (pos >> 3) + 8, 8);
    lo |= v << sh;
    if (sh) hi |= v >> (64 - sh);
    std::memcpy(dst + (pos >> 3), &lo, 8);
    std::memcpy(dst + (pos >> 3) + 8, &hi, 8);
}

// The flattened M^T of a descriptor (hmatrix.hpp:128 transpose = true): row and
// column ranges swap; a per-column lowrank leaf W Sigma X^H becomes X Sigma W^H
// and U V^T becomes V U^T (buffer order permuted, bytes shared); a dense leaf's
// column-major fields are re-ordered into the transposed block's column-major
// scan (every field keeps its bits; appended to the blob copy).
struct Transposed {
    std::vector<int64_t> row0, row1, col0, col1, count, poff, plen;
    std::vector<hcmx_descriptor> desc;
    std::vector<uint8_t> blob;
    hcmx_hmat_desc d{};
};

void make_transposed(const hcmx_hmat_desc& d, Transposed& t) {
    const uint64_t L = d.nleaves, nb = d.nbuffers;
    t.row0.assign(d.col0, d.col0 + L);
    t.row1.assign(d.col1, d.col1 + L);
    t.col0.assign(d.row0, d.row0 + L);
    t.col1.assign(d.row1, d.row1 + L);
    t.desc.assign(d.desc, d.desc + nb);
    t.count.assign(d.count, d.count + nb);
    t.poff.assign(d.poff, d.poff + nb);
    t.plen.assign(d.plen, d.plen + nb);
    uint64_t extra = 0;
    for (uint64_t l = 0; l < L; ++l)
        if (d.kind[l] == 0) extra += static_cast<uint64_t>(d.plen[d.buf0[l]]) + 16;
    t.blob.assign(d.blob_bytes + extra + 32, 0);
    if (d.blob_on_device)
        check_cuda(cudaMemcpy(t.blob.data(), d.blob, d.blob_bytes, cudaMemcpyDeviceToHost), "blob d2h");
    else
        std::memcpy(t.blob.data(), d.blob, d.blob_bytes);
    uint64_t at = (d.blob_bytes + 15) & ~uint64_t(15);
    auto take = [&](uint64_t dst, uint64_t src) {
        t.desc[dst] = d.desc[src];
        t.count[dst] = d.count[src];
        t.poff[dst] = d.poff[src];
        t.plen[dst] = d.plen[src];
    };
    for (uint64_t l = 0; l < L; ++l) {
        const uint64_t b0 = static_cast<uint64_t>(d.buf0[l]);
        const int64_t k = d.rank[l];
        if (d.kind[l] == 1) {
            for (int64_t i = 0; i < k; ++i) {
                take(b0 + i, b0 + k + i);
                take(b0 + k + i, b0 + i);
            }
        } else if (d.kind[l] == 2) {
            if (k > 0) {
                take(b0, b0 + 1);
                take(b0 + 1, b0);
            }
        } else {
            const uint64_t rows = d.row1[l] - d.row0[l], cols = d.col1[l] - d.col0[l];
            const unsigned w = d.desc[b0].bit_width;
            const uint8_t* src = t.blob.data() + d.poff[b0];
            uint8_t* dst = t.blob.data() + at;
            for (uint64_t c = 0; c < cols; ++c)
                for (uint64_t r = 0; r < rows; ++r)
                    put_field(dst, (c + r * cols) * w, w, get_field(src, (r + c * rows) * w, w));
            t.poff[b0] = static_cast<int64_t>(at);
            at += (static_cast<uint64_t>(d.plen[b0]) + 15) & ~uint64_t(15);
        }
    }
    t.d = d;
    t.d.n_rows = d.n_cols;
    t.d.n_cols = d.n_rows;
    t.d.row0 = t.row0.data();
    t.d.row1 = t.row1.data();
    t.d.col0 = t.col0.data();
    t.d.col1 = t.col1.data();
    t.d.desc = t.desc.data();
    t.d.count = t.count.data();
    t.d.poff = t.poff.data();
    t.d.plen = t.plen.data();
    t.d.blob = t.blob.data();
    t.d.blob_bytes = at;
    t.d.blob_on_device = 0;
    t.d.row_begin = t.d.row_end = 0;
    t.d.with_transpose = 0;
}

void destroy_handle(hcmx_hmat* h) {
    if (!h) return;
    destroy_handle(h->trans);
    destroy_handle(h->multi);
    if (h->stream) cudaStreamSynchronize(h->stream);
    for (auto& r : h->pending) {
        cudaEventDestroy(r.a0);
        cudaEventDestroy(r.a1);
        cudaEventDestroy(r.b1);
    }
    for (auto e : h->ev_pool) cudaEventDestroy(e);
    if (h->last) cudaEventDestroy(h->last);
    if (h->stream) cudaStreamDestroy(h->stream);
    delete h;
}

hcmx_hmat* create_handle(const hcmx_hmat_desc& d) {
    auto* h = new hcmx_hmat();
    try {
        check_cuda(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking), "cudaStreamCreate");
        if (d.complex_pairs) {
            // a complex matrix exists only as the 4-RHS arena (two complex columns per
            // product); the outer handle is a shell that forwards to it
            if (d.nrhs_block != kMultiR && d.nrhs_block != kMultiR2)
                throw invalid_argument("hmat: a complex matrix needs nrhs_block = 4 or 8");
            if (d.with_transpose || d.row_begin || d.row_end)
                throw invalid_argument("hmat: complex matrices: no transpose, no row partition");
            for (uint64_t l = 0; l < d.nleaves; ++l)
                if (d.kind[l] == 2) throw invalid_argument("hmat: complex matrices take APLR lowrank leaves (kind 1)");
            h->multi = new hcmx_hmat();
            h->multi->R = d.nrhs_block;
            h->multi->cplx = true;
            check_cuda(cudaStreamCreateWithFlags(&h->multi->stream, cudaStreamNonBlocking), "cudaStreamCreate");
            build(d, h->multi);
            h->cplx = true;
            h->n_rows = h->multi->n_rows;
            h->n_cols = h->multi->n_cols;
            h->rb = h->multi->rb;
            h->re = h->multi->re;
            h->report = h->multi->report;
            return h;
        }
        build(d, h);
        if (d.nrhs_block) {
            if (d.nrhs_block != kMultiR && d.nrhs_block != kMultiR2)
                throw invalid_argument("hmat: nrhs_block must be 0, 4 or 8");
            h->multi = new hcmx_hmat();
            h->multi->R = d.nrhs_block;
            check_cuda(cudaStreamCreateWithFlags(&h->multi->stream, cudaStreamNonBlocking), "cudaStreamCreate");
            build(d, h->multi);
        }
        if (d.with_transpose) {
            if (d.row_begin != 0 || d.row_end != 0)
                throw invalid_argument("hmat: the transpose needs the whole matrix (no row partition)");
            Transposed t;
            make_transposed(d, t);
            h->trans = create_handle(t.d);
        }
    } catch (...) {
        destroy_handle(h);
        throw;
    }
    return h;
}

}  // namespace

extern "C" {

int hcmx_gpu_hmat_create(const hcmx_hmat_desc* desc, hcmx_hmat** out) {
    return guarded([&] {
        require_device();
        *out = create_handle(*desc);
    });
}

int hcmx_gpu_hmat_transposed(hcmx_hmat* h, hcmx_hmat** out) {
    return guarded([&] {
        if (!h->trans) throw invalid_argument("hmat: created without with_transpose");
        *out = h->trans;
    });
}

int hcmx_gpu_hmat_destroy(hcmx_hmat* h) {
    return guarded([&] { destroy_handle(h); });
}

int hcmx_gpu_hmat_memory(const hcmx_hmat* h, hcmx_memory_report* out) {
    return guarded([&] { *out = h->report; });
}

int hcmx_gpu_hmat_matmat(hcmx_hmat* h, double alpha, const double* h_x, uint64_t ldx, uint64_t nrhs,
                         double beta, double* h_y, uint64_t ldy, int transpose) {
    return guarded([&] {
        if (h->cplx) throw invalid_argument("hmat: a complex matrix runs through hcmx_gpu_hmat_matmat4_device (two complex columns per product)");
        if (transpose) {
            if (!h->trans) throw invalid_argument("matmat: transpose needs a handle created with with_transpose");
            h = h->trans;
        }
        if (ldx < h->n_cols || ldy < h->n_rows) throw invalid_argument("matmat: leading dimension too small");
        if (!nrhs) return;
        if (h->multi && nrhs >= 2) {
            // blocks of nrhs_block columns through the multi-RHS arena: each field is
            // decoded once for the block (x and y interleaved n x nrhs_block; a short
            // last block is padded with zero columns)
            hcmx_hmat* mh = h->multi;
            const uint64_t B = static_cast<uint64_t>(mh->R);
            const uint64_t n = h->n_cols, nr = h->re - h->rb;
            DevBuf dx(n * B * 8), dy(h->n_rows * B * 8);
            std::vector<double> hx(n * B), hy(nr * B);
            for (uint64_t j0 = 0; j0 < nrhs; j0 += B) {
                const uint64_t cnt = std::min<uint64_t>(B, nrhs - j0);
                for (uint64_t i = 0; i < n; ++i)
                    for (uint64_t c = 0; c < B; ++c) hx[i * B + c] = c < cnt ? h_x[(j0 + c) * ldx + i] : 0.0;
                h2d(dx.p, hx.data(), n * B * 8, mh->stream);
                if (beta != 0.0) {
                    for (uint64_t i = 0; i < nr; ++i)
                        for (uint64_t c = 0; c < B; ++c) hy[i * B + c] = c < cnt ? h_y[(j0 + c) * ldy + h->rb + i] : 0.0;
                    h2d(dy.as<double>() + h->rb * B, hy.data(), nr * B * 8, mh->stream);
                }
                run_matvec(mh, alpha, dx.as<double>(), beta, dy.as<double>(), mh->stream);
                d2h(hy.data(), dy.as<double>() + h->rb * B, nr * B * 8, mh->stream);
                stream_sync(mh->stream);
                for (uint64_t i = 0; i < nr; ++i)
                    for (uint64_t c = 0; c < cnt; ++c) h_y[(j0 + c) * ldy + h->rb + i] = hy[i * B + c];
            }
            return;
        }
        // all right-hand sides in one copy each way; one product per column
        DevBuf dx(h->n_cols * nrhs * 8), dy(h->n_rows * nrhs * 8);
        for (uint64_t j = 0; j < nrhs; ++j) h2d(dx.as<double>() + j * h->n_cols, h_x + j * ldx, h->n_cols * 8, h->stream);
        const uint64_t nr = h->re - h->rb;
        if (beta != 0.0)
            for (uint64_t j = 0; j < nrhs; ++j)
                h2d(dy.as<double>() + j * h->n_rows + h->rb, h_y + j * ldy + h->rb, nr * 8, h->stream);
        for (uint64_t j = 0; j < nrhs; ++j)
            run_matvec(h, alpha, dx.as<double>() + j * h->n_cols, beta, dy.as<double>() + j * h->n_rows, h->stream);
        for (uint64_t j = 0; j < nrhs; ++j) d2h(h_y + j * ldy + h->rb, dy.as<double>() + j * h->n_rows + h->rb, nr * 8, h->stream);
        stream_sync(h->stream);
    });
}

int hcmx_gpu_hmat_matvec_device(hcmx_hmat* h, double alpha, const double* d_x, double beta, double* d_y,
                                void* stream) {
    return guarded([&] {
        if (h->cplx) throw invalid_argument("hmat: a complex matrix runs through hcmx_gpu_hmat_matmat4_device (two complex columns per product)");
        run_matvec(h, alpha, d_x, beta, d_y, (cudaStream_t)stream);
    });
}

int hcmx_gpu_hmat_matmat4_device(hcmx_hmat* h, double alpha, const double* d_x4, double beta, double* d_y4,
                                 void* stream) {
    return guarded([&] {
        if (!h->multi) throw invalid_argument("matmat4: handle created without nrhs_block = 4");
        if (h->multi->R != kMultiR) throw invalid_argument("matmat4: handle built with nrhs_block = 8 (use matmat_block_device)");
        if (reinterpret_cast<uintptr_t>(d_x4) % 16) throw invalid_argument("matmat4: x must be 16-byte aligned");
        run_matvec(h->multi, alpha, d_x4, beta, d_y4, (cudaStream_t)stream);
    });
}

int hcmx_gpu_hmat_matmat_block_device(hcmx_hmat* h, double alpha, const double* d_x, double beta, double* d_y,
                                      void* stream) {
    return guarded([&] {
        if (!h->multi) throw invalid_argument("matmat_block: handle created without nrhs_block");
        if (reinterpret_cast<uintptr_t>(d_x) % 16) throw invalid_argument("matmat_block: x must be 16-byte aligned");
        run_matvec(h->multi, alpha, d_x, beta, d_y, (cudaStream_t)stream);
    });
}

int hcmx_gpu_hmat_nrhs_block(const hcmx_hmat* h) { return h && h->multi ? h->multi->R : 0; }

int hcmx_gpu_hmat_matvec(hcmx_hmat* h, double alpha, const double* h_x, double beta, double* h_y,
                         int transpose) {
    return guarded([&] {
        if (h->cplx) throw invalid_argument("hmat: a complex matrix runs through hcmx_gpu_hmat_matmat4_device (two complex columns per product)");
        if (transpose) {  // hmatrix.hpp:128: y (n_cols) := alpha M^T x + beta y
            if (!h->trans) throw invalid_argument("matvec: transpose needs a handle created with with_transpose");
            h = h->trans;
        }
        std::lock_guard<std::mutex> io(h->io_mu);
        if (!h->xbuf.p) h->xbuf.alloc(h->n_cols * 8);
        const uint64_t nr = h->re - h->rb;
        h2d(h->xbuf.p, h_x, h->n_cols * 8, h->stream);
        // y in pinned (page-locked, device-mapped) host memory: the kernels write
        // the rows straight into it over PCIe while phase B runs -- no device
        // staging and no copy back after the product (x is read many times, so it
        // is always staged in HBM)
        static const bool no_mapped = std::getenv("HCMX_NO_MAPPED_Y") != nullptr;  // A/B knob
        cudaPointerAttributes pa{};
        const bool mapped = !no_mapped && beta == 0.0 && cudaPointerGetAttributes(&pa, h_y) == cudaSuccess &&
                            pa.type == cudaMemoryTypeHost && pa.devicePointer != nullptr;
        cudaGetLastError();  // a pageable pointer may leave an error flag behind
        if (mapped) {
            run_matvec(h, alpha, h->xbuf.as<double>(), beta, static_cast<double*>(pa.devicePointer), h->stream);
            stream_sync(h->stream);
            return;
        }
        if (!h->ybuf.p) h->ybuf.alloc(h->n_rows * 8);
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
        std::vector<uint8_t> bits(((n + 16) & ~uint64_t(3)) + 16, 0);
        for (const SegRef& sref : h->segs[b]) {
            const uint64_t nbits = sref.gwords ? static_cast<uint64_t>((sref.nf + kARows - 1) / kARows) * sref.gwords * 32
                                               : static_cast<uint64_t>(sref.nf) * w;
            const uint64_t nw = (nbits + 31) / 32;
            std::vector<uint32_t> words(nw + 2, 0u);
            check_cuda(cudaMemcpy(words.data(), h->arena.as<uint32_t>() + sref.word, nw * 4, cudaMemcpyDeviceToHost),
                       "export d2h");
            for (uint64_t j = 0; j < sref.nf; ++j) {
                // the field in the arena run, written back at its original offset
                const FieldLoc fl = field_loc(sref, j, w);
                put_bits(reinterpret_cast<uint32_t*>(bits.data()), (sref.f0 + j) * w,
                         get_bits_strided(words.data() + fl.word, words.size() - fl.word, fl.stride, fl.bit, w), w);
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
