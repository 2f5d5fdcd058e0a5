/*
 * hcmx_gpu.h -- C-ABI of the B200 (sm_100a) implementation of the hcmx hot path:
 * the adaptive-precision codec (AFL/AFLP/BFL/DFL), APLR per-column lowrank
 * compression and the compressed H-matrix-vector product.
 *
 * Every entry point replaces a function of the reference C++ API in
 * /root/reference/proj/include/hcmx (cited per function).  The reference has no
 * FFI; the binding a maintainer adds is shown in INTEGRATION.md (a C++ shim
 * keeping the hcmx::codec / hcmx::matvec names, and a ctypes stub).
 *
 * Conventions
 *   - plain pointers and sizes, no C++ or torch types; "d_" = device pointer,
 *     "h_" = host pointer.  Streams are cudaStream_t passed as void*.
 *   - every function returns HCMX_OK (0) or an error status; the reference's
 *     exceptions map to statuses: std::invalid_argument -> HCMX_INVALID_ARGUMENT,
 *     hcmx::corrupt_buffer_error (common.hpp:17-19) -> HCMX_CORRUPT_BUFFER.
 *     hcmx_gpu_last_error() returns the message of the last failure on the
 *     calling thread.
 *   - there is no CPU fallback: without a usable sm_100 device every compute
 *     entry point returns HCMX_CUDA_ERROR.
 */
#ifndef HCMX_GPU_H
#define HCMX_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum hcmx_status {
    HCMX_OK = 0,
    HCMX_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    HCMX_CORRUPT_BUFFER = 2,   /* hcmx::corrupt_buffer_error */
    HCMX_CUDA_ERROR = 3,
    HCMX_NCCL_ERROR = 4,
    HCMX_OUT_OF_MEMORY = 5
};

/* codec::Scheme (codec.hpp:22).  The matvec also accepts buffers of uncompressed
 * IEEE words (StorageMode fp64, hmatrix.hpp:32-40, and the FP64/FP32/FP16 groups
 * of mp::MPLowrank, mixedprec.hpp:20-43): bit_width 64/32/16, scale 1.  The codec
 * entry points reject these. */
enum hcmx_scheme {
    HCMX_AFL = 0, HCMX_AFLP = 1, HCMX_BFL = 2, HCMX_DFL = 3,
    HCMX_RAW_F64 = 4, HCMX_RAW_F32 = 5, HCMX_RAW_F16 = 6
};

/* codec::FormatDescriptor (codec.hpp:35-56), 16 bytes */
typedef struct hcmx_descriptor {
    uint8_t scheme;
    uint8_t exp_bits;
    uint8_t mant_bits;
    uint8_t bit_width; /* cached FormatDescriptor::bit_width() */
    uint32_t reserved;
    double scale;
} hcmx_descriptor;

/* codec::BlockStats (codec.hpp:68-72) + a non-finite flag, 24 bytes */
typedef struct hcmx_stats {
    double min_mag;
    double max_mag;
    uint32_t all_zero;
    uint32_t non_finite; /* compress rejects these (codec.cpp:119-120) */
} hcmx_stats;

/* ---------------------------------------------------------------- setup -- */
int hcmx_gpu_init(int device);
const char* hcmx_gpu_last_error(void);
int hcmx_gpu_version(void);

/* ----------------------------------------- scalar layout rules (host) ---- */
/* codec.cpp:62-67 */
int hcmx_gpu_mantissa_bits_for(double eps, uint8_t* out);
/* codec.cpp:69-79 */
int hcmx_gpu_exponent_bits_for(const hcmx_stats* stats, uint8_t* out);
/* codec.cpp:81-84: make_descriptor(scheme, eps, stats) */
int hcmx_gpu_make_descriptor(int scheme, double eps, const hcmx_stats* stats, hcmx_descriptor* out);
/* codec.cpp:86-101: make_descriptor(scheme, eps, scale, exp_bits) */
int hcmx_gpu_make_descriptor_pinned(int scheme, double eps, double scale, uint8_t exp_bits,
                                    hcmx_descriptor* out);
/* codec.hpp:51-55 */
unsigned hcmx_gpu_bit_width(const hcmx_descriptor* d);
/* codec.cpp:179-181 (20-byte header + packed payload) */
uint64_t hcmx_gpu_compressed_size(uint64_t count, const hcmx_descriptor* d);
/* payload bytes only: ceil(count * bit_width / 8) */
uint64_t hcmx_gpu_payload_bytes(uint64_t count, const hcmx_descriptor* d);

/* ------------------------------------------- batched device codec -------- */
/* A batch is nbuf independent buffers; buffer b holds h_count[b] FP64 values
 * at d_values + d_voff[b] (element offsets) and its packed payload at
 * d_payload + d_poff[b] (byte offsets, 16-byte aligned; each slot must hold
 * round_up(payload_bytes, 16) bytes).  Packed payloads are byte-for-byte the
 * reference's CompressedBuffer::payload.  h_count is a HOST array: the library
 * splits big buffers into warp jobs of <= 16384 values on the host. */

/* codec.cpp:44-60 analyze, one hcmx_stats per buffer (warp-shuffle min/max) */
int hcmx_gpu_codec_analyze(const double* d_values, const uint64_t* d_voff, const uint64_t* h_count,
                           uint64_t nbuf, hcmx_stats* d_stats, void* stream);

/* codec.cpp:103-140 compress_block for every buffer with caller-pinned layouts */
int hcmx_gpu_codec_pack(const double* d_values, const uint64_t* d_voff, const uint64_t* h_count,
                        const hcmx_descriptor* d_desc, const uint64_t* d_poff, uint64_t nbuf,
                        uint8_t* d_payload, void* stream);

/* codec.cpp:146-171 decompress_into for every buffer */
int hcmx_gpu_codec_unpack(const uint8_t* d_payload, const uint64_t* d_poff, const uint64_t* h_count,
                          const hcmx_descriptor* d_desc, const uint64_t* d_voff, uint64_t nbuf,
                          double* d_out, void* stream);

/* codec.cpp:142-144 compress for every buffer: analyze on the device, layout
 * selection on the host with the reference's exact scalar rules (glibc log2),
 * payload offsets (16-byte aligned) and packing on the device.  Outputs h_desc[nbuf], h_poff[nbuf] and *h_total
 * (arena bytes used); fails with HCMX_INVALID_ARGUMENT on non-finite input or
 * eps outside (0,1), and if the arena capacity is too small. */
int hcmx_gpu_codec_compress(const double* d_values, const uint64_t* d_voff,
                            const uint64_t* h_count, uint64_t nbuf, double eps, int scheme,
                            uint8_t* d_payload, uint64_t payload_capacity, hcmx_descriptor* h_desc,
                            uint64_t* h_poff, uint64_t* h_total, void* stream);

/* codec.cpp:142-144 compress for a batch with everything on the device and no
 * host synchronisation (no per-call read-back): counts d_count (each <=
 * max_count <= 2^17 values), caller-sized payload slots at d_poff (16-byte
 * aligned; a slot must hold the widest layout the scheme allows, exp_bits 11),
 * descriptors to d_desc and per-buffer flags to d_flags: bit 0 = the exponent
 * width was decided next to a 2^k - 2 threshold with the device log2 (the
 * reference decides it with glibc, codec.cpp:72-73) -- run
 * hcmx_gpu_codec_compress_fixup before trusting such a buffer; bit 1 =
 * non-finite input (that buffer is not packed; codec.cpp:119-120). */
int hcmx_gpu_codec_compress_device(const double* d_values, const uint64_t* d_voff, const uint64_t* d_count,
                                   uint64_t nbuf, uint64_t max_count, double eps, int scheme,
                                   const uint64_t* d_poff, uint8_t* d_payload, hcmx_descriptor* d_desc,
                                   uint32_t* d_flags, void* stream);
/* completes a compress_device batch bit-exactly: reads the flags (synchronises),
 * re-decides every flagged exponent width with the reference's host rule and
 * repacks those buffers; HCMX_INVALID_ARGUMENT if any input was non-finite.
 * *n_fixed = buffers whose layout changed. */
int hcmx_gpu_codec_compress_fixup(const double* d_values, const uint64_t* d_voff, const uint64_t* h_count,
                                  uint64_t nbuf, double eps, int scheme, const uint64_t* h_poff,
                                  uint8_t* d_payload, hcmx_descriptor* d_desc, const uint32_t* d_flags,
                                  uint64_t* n_fixed, void* stream);

/* Device time of the batched codec kernels (CUDA events around the fused compress
 * and the unpack launches), accumulated since the last reset.  enable: 1 on, 0 off,
 * < 0 query only (no reset).  Instrumentation for the benchmark, not a reference API. */
int hcmx_gpu_codec_timing(int enable, double* ms_compress, uint64_t* n_compress, double* ms_decompress,
                          uint64_t* n_decompress);

/* Single-buffer, HOST-pointer forms of codec::compress / decompress_into
 * (codec.cpp:142-171): the reference-facing call.  Copies in, runs the device
 * kernels, copies out. */
int hcmx_gpu_compress(const double* h_values, uint64_t count, double eps, int scheme,
                      hcmx_descriptor* desc, uint8_t* h_payload, uint64_t capacity,
                      uint64_t* payload_len);
int hcmx_gpu_compress_block(const double* h_values, uint64_t count, const hcmx_descriptor* desc,
                            uint8_t* h_payload, uint64_t capacity, uint64_t* payload_len);
int hcmx_gpu_decompress_into(const hcmx_descriptor* desc, uint64_t count, const uint8_t* h_payload,
                             uint64_t payload_len, double* h_out);

/* codec.cpp:187-225 wire format [u8 scheme][u8 e][u8 m][u8 0][f64 scale][u64 count][payload] */
uint64_t hcmx_gpu_serialize(const hcmx_descriptor* desc, uint64_t count, const uint8_t* payload,
                            uint64_t payload_len, uint8_t* out);
int hcmx_gpu_deserialize(const uint8_t* data, uint64_t size, uint64_t* offset,
                         hcmx_descriptor* desc, uint64_t* count, uint64_t* payload_at,
                         uint64_t* payload_len);

/* ------------------------------------------------------------- APLR ------ */
/* mixedprec.cpp:155-187 aplr_compress for a batch of lowrank leaves from given
 * factors: leaf j has W (rows_j x k_j) and X (cols_j x k_j) column-major at
 * d_W + h_woff[j], d_X + h_xoff[j] and sigma at h_sigma + h_soff[j].  Column i of
 * W becomes buffer h_boff[j] + i, column i of X buffer h_boff[j] + k_j + i.
 * e is analysed over the whole factor, per column eps_i = min(0.5, eps sigma_0 /
 * sigma_i) and scale = column min |v|.  Outputs descriptors / 16-byte-aligned
 * payload offsets for all buffers. */
int hcmx_gpu_aplr_compress(uint64_t nleaves, const uint64_t* h_rows, const uint64_t* h_cols,
                           const uint64_t* h_k, const double* d_W, const uint64_t* h_woff,
                           const double* d_X, const uint64_t* h_xoff, const double* h_sigma,
                           const uint64_t* h_soff, const uint64_t* h_boff, double eps, int scheme,
                           uint8_t* d_payload, uint64_t payload_capacity, hcmx_descriptor* h_desc,
                           uint64_t* h_poff, uint64_t* h_total, void* stream);

/* ------------------------------------------------------- H-matrix -------- */
/* Flattened H-matrix (hmatrix.hpp:51-78): leaves in for_each_leaf preorder
 * (clustering.cpp:159-166, children row-major 2i+j), internal index space.
 *   kind 0 CodecDense  (hmatrix.hpp:42-44): buffer buf0, column-major scan
 *   kind 1 APLRLowrank (mixedprec.hpp:68-82): buffers buf0..buf0+k-1 = W columns,
 *          buf0+k..buf0+2k-1 = X columns, sigma[sig0 .. sig0+k).  With raw FP64 /
 *          FP32 / FP16 column buffers the same kind holds mp::MPLowrank
 *          (mixedprec.hpp:46-64: W Sigma X^H, columns grouped by format).
 *   kind 2 CodecLowrank (hmatrix.hpp:46-49) / LowrankBlock (lowrank.hpp:17-29):
 *          buffer buf0 = U (rows x k, column-major), buf0+1 = V (cols x k),
 *          y += U (V^T x); codec-compressed or raw FP64 words
 * Buffers: descriptor, value count, payload at blob[poff .. poff+plen). */
typedef struct hcmx_hmat_desc {
    uint64_t n_rows, n_cols, nleaves, nbuffers, nsigma, blob_bytes;
    const int64_t *row0, *row1, *col0, *col1, *kind, *rank, *buf0, *sig0; /* [nleaves] */
    const double* sigma;                                                  /* [nsigma] */
    const hcmx_descriptor* desc;                                          /* [nbuffers] */
    const int64_t *count, *poff, *plen;                                   /* [nbuffers] */
    const uint8_t* blob; /* host pointer, or device pointer if blob_on_device */
    int blob_on_device;
    /* block-row partition (multi-GPU): every leaf that overlaps [row_begin,row_end)
     * is loaded (a lowrank leaf crossing the range boundary does its X^T x half
     * here too); matvec then writes y[row_begin,row_end) only. 0,0 = all rows */
    uint64_t row_begin, row_end;
    /* nonzero: also build M^T (hmatrix.hpp:128 transpose; whole matrix only) */
    int with_transpose;
    /* 4 or 8: also lay the matrix out for products with 4 / 8 right-hand sides
     * at once (hcmx_gpu_hmat_matmat decodes every field once per block of
     * nrhs_block columns); 0: off */
    int nrhs_block;
    /* nonzero: a COMPLEX matrix A = Ar + i Ai stored once with real codec streams
     * (BASELINE config 5; needs nrhs_block = 4 or 8, no transpose).  Lowrank leaves
     * (kind 1) hold A's truncated SVD U S V^H as W = [Ur Ui], X = [Vr Vi] and
     * sigma = [S S] (rank 2k: every real / imaginary factor column is its own
     * APLR stream, decoded once per product); dense leaves are Re A (imag 0) and
     * Im A (dense_imag[l] = 1, same row / column range).  The block products then
     * take nrhs_block / 2 complex columns interleaved, [Re x1, Im x1, Re x2, ...],
     * and return [Re y1, Im y1, Re y2, ...]; the complex combination of the
     * X^T x halves runs on the device between the phases. */
    int complex_pairs;
    const uint8_t* dense_imag; /* [nleaves], or NULL */
} hcmx_hmat_desc;

typedef struct hcmx_hmat hcmx_hmat; /* opaque, device resident */

/* MemoryReport (hmatrix.hpp:96-113) + device arena accounting */
typedef struct hcmx_memory_report {
    uint64_t dense_raw, dense_compressed, lowrank_raw, lowrank_compressed, overhead;
    uint64_t uncompressed_equivalent;
    uint64_t device_arena_bytes;   /* packed streams resident in HBM */
    uint64_t device_table_bytes;   /* stage / item / column tables */
    uint64_t algorithmic_bytes;    /* bytes one matvec must move */
    uint64_t dense_leaves, lowrank_leaves, stages_a, stages_b;
} hcmx_memory_report;

/* ------------------------------------------------- compress_in_place ----- */
/* An assembled, uncompressed H-matrix (the input of compress_in_place,
 * hmatrix.hpp:115-119): leaf ranges on the host; FP64 payloads on the device.
 *   kind 0 dense leaf: rows x cols column-major at d_dense + dense_off[l]
 *   kind 1 lowrank leaf W diag(sigma) X^T (svd_factors' shape, lowrank.cpp:76-93):
 *          W rows x k column-major at d_W + w_off[l], X cols x k at d_X + x_off[l],
 *          sigma[sig_off[l] .. + k) on the host */
typedef struct hcmx_assembled {
    uint64_t n_rows, n_cols, nleaves;
    const int64_t *row0, *row1, *col0, *col1, *kind, *rank; /* [nleaves], host */
    const double* d_dense;
    const int64_t* dense_off;
    const double *d_W, *d_X;
    const int64_t *w_off, *x_off;
    const double* sigma;
    const int64_t* sig_off;
} hcmx_assembled;

/* StorageMode kinds (hmatrix.hpp:32-40) */
enum hcmx_storage { HCMX_STORE_APLR = 0, HCMX_STORE_CODEC = 1, HCMX_STORE_MP = 2, HCMX_STORE_FP64 = 3 };

typedef struct hcmx_flat hcmx_flat; /* a compressed, flattened H-matrix: host tables + device blob */

/* compress_in_place (hmatrix.hpp:115-119) on the device:
 *   APLR   dense -> codec::compress iff dense_too (else FP64 words); lowrank ->
 *          APLR (per-column precision from sigma, mixedprec.cpp:155-187)
 *   CODEC  dense as above; lowrank U = W diag(sigma), V = X as one codec buffer
 *          each (CodecLowrank, hmatrix.hpp:46-49)
 *   MP     dense FP64; lowrank columns in FP64 / FP32 / FP16 groups
 *          (mp_partition, mixedprec.cpp:66-120)
 *   FP64   uncompressed (dense FP64, U and V FP64)
 * Bytes equal the reference codec's (tests).  *report = memory_footprint
 * (hmatrix.hpp:96-124) of the result. */
int hcmx_gpu_compress_in_place(const hcmx_assembled* A, double eps, int storage, int scheme, int dense_too,
                               hcmx_flat** out, hcmx_memory_report* report, void* stream);
/* the result as an hcmx_hmat_desc (pointers into f, blob_on_device = 1), ready
 * for hcmx_gpu_hmat_create / _create_partitioned; valid while f lives */
int hcmx_gpu_flat_desc(const hcmx_flat* f, hcmx_hmat_desc* desc);
/* copies the device blob (desc.blob_bytes) into caller device memory */
int hcmx_gpu_flat_copy_blob(const hcmx_flat* f, uint8_t* d_dst, void* stream);
int hcmx_gpu_flat_destroy(hcmx_flat* f);

int hcmx_gpu_hmat_create(const hcmx_hmat_desc* desc, hcmx_hmat** out);
int hcmx_gpu_hmat_destroy(hcmx_hmat* h);
int hcmx_gpu_hmat_memory(const hcmx_hmat* h, hcmx_memory_report* out);

/* hmatrix.hpp:126-128 matvec: y := alpha * M * x + beta * y (beta == 0 overwrites
 * y; alpha == 0 gives beta * y without touching M).  Host-pointer form: copies x in
 * and y out (the reference-facing call).  transpose != 0: y (n_cols) := alpha M^T x
 * + beta y, for handles created with with_transpose (else HCMX_INVALID_ARGUMENT). */
int hcmx_gpu_hmat_matvec(hcmx_hmat* h, double alpha, const double* h_x, double beta, double* h_y,
                         int transpose);
/* several right-hand sides: Y := alpha op(M) X +
 * beta Y for nrhs host columns (column-major, leading dimensions ldx / ldy).  A
 * handle created with nrhs_block = 4 runs blocks of 4 columns through its 4-RHS
 * arena (every field decoded once per block, a short last block padded with
 * zero columns); otherwise one device product per column. */
int hcmx_gpu_hmat_matmat(hcmx_hmat* h, double alpha, const double* h_x, uint64_t ldx, uint64_t nrhs,
                         double beta, double* h_y, uint64_t ldy, int transpose);
/* device-pointer form on a stream; d_x has n_cols entries, d_y n_rows entries
 * (for a partitioned handle only d_y[row_begin,row_end) is written).  Products
 * on one handle share its device scratch: a product issued on another stream
 * than the handle's previous one waits for that product first (an event), so
 * one handle may be used from several streams and host threads. */
int hcmx_gpu_hmat_matvec_device(hcmx_hmat* h, double alpha, const double* d_x, double beta,
                                double* d_y, void* stream);

/* Four right-hand sides at once through the multi-RHS arena (handles created
 * with nrhs_block = 4): Y := alpha M X + beta Y with X (n_cols x 4) and Y
 * (n_rows x 4) ROW-major on the device (the 4 columns interleaved), every
 * packed field decoded once for the 4 columns.  Same stream rules as
 * hcmx_gpu_hmat_matvec_device.  C5's multi-RHS products. */
int hcmx_gpu_hmat_matmat4_device(hcmx_hmat* h, double alpha, const double* d_x4, double beta, double* d_y4,
                                 void* stream);
/* the same with the handle's nrhs_block (4 or 8) columns interleaved: x is
 * n_cols x nrhs_block, y n_rows x nrhs_block, row-major, 16-byte aligned */
int hcmx_gpu_hmat_matmat_block_device(hcmx_hmat* h, double alpha, const double* d_x, double beta,
                                      double* d_y, void* stream);
/* the right-hand sides per product of the handle's multi-RHS arena (0: none) */
int hcmx_gpu_hmat_nrhs_block(const hcmx_hmat* h);

/* the handle of M^T inside a handle created with with_transpose (owned by h;
 * use it with the _device / _timing calls) */
int hcmx_gpu_hmat_transposed(hcmx_hmat* h, hcmx_hmat** out);

/* rebuild buffer b's verbatim payload from the device arena (layout check) */
int hcmx_gpu_hmat_export_buffer(const hcmx_hmat* h, uint64_t b, uint8_t* h_payload,
                                uint64_t capacity, uint64_t* len);

/* launch counting for the bench: kernels launched by the last matvec */
int hcmx_gpu_hmat_last_launches(const hcmx_hmat* h);

/* per-kernel device timing of the hot kernels (CUDA events on the launch
 * stream) accumulated over matvec_device calls since the last reset */
int hcmx_gpu_hmat_timing(hcmx_hmat* h, int enable, double* ms_phase_a, double* ms_phase_b,
                         uint64_t* calls);

/* ------------------------------------------- block-row partitions (multi-GPU) */
/* the rows are cut into one contiguous range per rank; each rank
 * keeps the leaves that write its rows, x is replicated and y slices are
 * disjoint, so the only exchange per product is an all-gather of y.  The
 * reference has no parallel code (its hooks: the unused `threads` knobs,
 * hmatrix.hpp:83,119, and SPEC.md:489's deterministic merge of disjoint leaf
 * blocks); y here is bit-identical to the single-GPU product. */

/* the partitioner: world + 1 cuts (multiples of 64 rows, cuts[world] = n_rows)
 * minimising the largest per-rank byte count, where a lowrank leaf crossing a
 * cut charges its X factor to both ranks.  Host only (no device needed). */
int hcmx_gpu_partition_rows(const hcmx_hmat_desc* desc, int world, uint64_t* cuts);

/* NCCL communicator helpers (libnccl.so.2 is loaded at run time; a caller that
 * already has an ncclComm_t passes it directly).  id128 = ncclUniqueId bytes. */
struct ncclComm; /* ncclComm_t == struct ncclComm* (nccl.h) */
int hcmx_gpu_nccl_unique_id(uint8_t* id128);
int hcmx_gpu_nccl_comm_init(int world, const uint8_t* id128, int rank, struct ncclComm** comm);
int hcmx_gpu_nccl_comm_destroy(struct ncclComm* comm);

typedef struct hcmx_hmat_dist hcmx_hmat_dist; /* this rank's rows + the communicator */
/* every rank passes the whole flattened matrix and the same communicator
 * (world and rank are taken from it; comm == NULL: one rank).  The handle is
 * built for hcmx_gpu_partition_rows' range of this rank (row_begin / row_end /
 * with_transpose of desc are ignored). */
int hcmx_gpu_hmat_create_partitioned(const hcmx_hmat_desc* desc, struct ncclComm* comm, hcmx_hmat_dist** out);
int hcmx_gpu_hmat_dist_destroy(hcmx_hmat_dist* h);
int hcmx_gpu_hmat_dist_rows(const hcmx_hmat_dist* h, uint64_t* row_begin, uint64_t* row_end, int* rank,
                            int* world);
int hcmx_gpu_hmat_dist_cuts(const hcmx_hmat_dist* h, uint64_t* cuts); /* world + 1 entries */
/* the rank-local handle (NULL for an empty range), for timing / memory queries */
int hcmx_gpu_hmat_dist_local(hcmx_hmat_dist* h, hcmx_hmat** local);
/* y := alpha M x + beta y on every rank: the local product of this rank's rows,
 * then one NCCL group of in-place broadcasts (rank r sends y[cut_r, cut_r+1))
 * on `stream`, so every rank ends with the whole contiguous y (n_rows) for the
 * next product.  x and y must be identical on all ranks.  NCCL failures ->
 * HCMX_NCCL_ERROR. */
int hcmx_gpu_hmat_dist_matvec_device(hcmx_hmat_dist* h, double alpha, const double* d_x, double beta,
                                     double* d_y, void* stream);
/* the same with host vectors (copies x in and the whole y out; the
 * reference-facing call of a partitioned matrix, hmatrix.hpp:126-128) */
int hcmx_gpu_hmat_dist_matvec(hcmx_hmat_dist* h, double alpha, const double* h_x, double beta, double* h_y);

#ifdef __cplusplus
}
#endif

#endif /* HCMX_GPU_H */
