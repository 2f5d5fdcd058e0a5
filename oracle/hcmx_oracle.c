/*
 * hcmx_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * A plain-C restatement of the reference hcmx codec, APLR glue and the
 * (declared-only) compressed H-matrix-vector product.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library.  The product path (paper_2308_10960_b200) never
 * links or calls it.
 *
 * Parity pin: tests/test_oracle.py checks every function below against the
 * reference codec compiled from /root/reference (oracle/_ref, built by
 * oracle/Makefile) and against the committed fixtures in tests/golden/.
 *
 * Build (oracle/Makefile): gcc -std=c11 -O2 -ffp-contract=off -fPIC -shared.
 * -ffp-contract=off matters: the reference's Release build emits a separate
 * multiply and add at codec.cpp:124; an FMA changes packed bytes.
 *
 * Citations are /root/reference/proj/... file:line.
 */
#define _GNU_SOURCE
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_INVALID_ARGUMENT 1
#define ORC_CORRUPT_BUFFER 2

enum { AFL = 0, AFLP = 1, BFL = 2, DFL = 3 };

static uint64_t dbits(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }
static double bitsd(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }

/* ---------------------------------------------------------------- RNG ---- */
/* std::mt19937_64 restated (used by proj/tests/oracles.hpp:57-70 Rng). */
typedef struct { uint64_t mt[312]; int idx; } orc_mt64;

void orc_mt64_seed(orc_mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

uint64_t orc_mt64_next(orc_mt64* g) {
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ull) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFull);
            uint64_t xa = x >> 1;
            if (x & 1ull) xa ^= 0xB5026F5AA96619E9ull;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t x = g->mt[g->idx++];
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= (x >> 43);
    return x;
}

/* raw 64-bit outputs of mt19937_64(seed) */
void orc_mt64_raw(uint64_t seed, int64_t n, uint64_t* out) {
    orc_mt64 g; orc_mt64_seed(&g, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = orc_mt64_next(&g);
}

/* oracles.hpp:60 uniform() = (g() >> 11) * 2^-53 */
static double orc_u01(orc_mt64* g) { return (double)(orc_mt64_next(g) >> 11) * 0x1.0p-53; }

/* oracles.hpp:64-67 log_uniform_signed, n values from one stream */
void orc_log_uniform_signed(uint64_t seed, int64_t n, double lo, double hi, double* out) {
    orc_mt64 g; orc_mt64_seed(&g, seed);
    for (int64_t i = 0; i < n; ++i) {
        double a = log(lo), b = log(hi);
        double mag = exp(a + (b - a) * orc_u01(&g));
        out[i] = orc_u01(&g) < 0.5 ? -mag : mag;
    }
}

/* BASELINE config 2 entries: sign * 10^U[-6,0] (sign uniform +-1) */
void orc_config2_values(uint64_t seed, int64_t n, double* out) {
    orc_mt64 g; orc_mt64_seed(&g, seed);
    for (int64_t i = 0; i < n; ++i) {
        double ex = -6.0 + 6.0 * orc_u01(&g);
        double mag = pow(10.0, ex);
        out[i] = orc_u01(&g) < 0.5 ? -mag : mag;
    }
}

/* ----------------------------------------------------- codec: layout ---- */
/* codec.hpp:40-49 alignment_unit */
static unsigned unit_of(int scheme) {
    switch (scheme) {
        case AFL: return 1;
        case AFLP: case BFL: return 8;
        case DFL: return 16;
    }
    return 1;
}

/* codec.hpp:51-55 bit_width */
int orc_bit_width(int scheme, int e, int m) {
    unsigned unit = unit_of(scheme);
    unsigned w = 1u + (unsigned)e + (unsigned)m;
    return (int)(w + (unit - w % unit) % unit);
}

/* codec.cpp:44-60 analyze */
void orc_analyze(const double* v, int64_t n, double* min_mag, double* max_mag, int* all_zero) {
    double mn = INFINITY, mx = 0.0;
    int az = 1;
    for (int64_t i = 0; i < n; ++i) {
        double a = fabs(v[i]);
        if (a == 0.0) continue;
        az = 0;
        mn = a < mn ? a : mn;   /* std::min(st.min_mag, a) */
        mx = mx < a ? a : mx;   /* std::max(st.max_mag, a) */
    }
    if (az) { mn = 0.0; mx = 0.0; }
    *min_mag = mn; *max_mag = mx; *all_zero = az;
}

static double clampd(double x, double lo, double hi) { return x < lo ? lo : (hi < x ? hi : x); }

/* codec.cpp:62-67 mantissa_bits_for */
int orc_mantissa_bits_for(double eps, int* out) {
    if (!(eps > 0.0) || !(eps < 1.0)) return ORC_INVALID_ARGUMENT;
    double bits = ceil(-log2(eps)) - 1.0;
    *out = (int)(uint8_t)clampd(bits, 2.0, 52.0);
    return ORC_OK;
}

/* codec.cpp:69-75 exponent_bits_for(BlockStats) */
int orc_exponent_bits_for_stats(double min_mag, double max_mag, int all_zero) {
    if (all_zero) return 2;
    double span = log2(max_mag) - log2(min_mag) + 1.0;
    double bits = ceil(log2(span + 1.0));
    return (int)(uint8_t)clampd(bits, 2.0, 11.0);
}

/* codec.cpp:77-79 exponent_bits_for(span) */
int orc_exponent_bits_for(const double* v, int64_t n) {
    double mn, mx; int az;
    orc_analyze(v, n, &mn, &mx, &az);
    return orc_exponent_bits_for_stats(mn, mx, az);
}

/* codec.cpp:25-30 align_mantissa */
static int align_mantissa(int scheme, int e, int m) {
    unsigned unit = unit_of(scheme);
    unsigned w = 1u + (unsigned)e + (unsigned)m;
    w += (unit - w % unit) % unit;
    unsigned r = w - 1u - (unsigned)e;
    return (int)(r < 52u ? r : 52u);
}

/* codec.cpp:86-101 make_descriptor(scheme, eps, scale, exp_bits) */
int orc_make_descriptor(int scheme, double eps, int exp_bits, int* e_out, int* m_out) {
    int e = exp_bits, m;
    if (scheme == BFL) e = 8;
    else if (scheme == DFL) e = 11;
    int st = orc_mantissa_bits_for(eps, &m);
    if (st) return st;
    if (scheme != AFL) m = align_mantissa(scheme, e, m);
    *e_out = e; *m_out = m;
    return ORC_OK;
}

/* codec.cpp:179-181 compressed_size */
int64_t orc_compressed_size(int64_t count, int scheme, int e, int m) {
    return 20 + (count * (int64_t)orc_bit_width(scheme, e, m) + 7) / 8;
}

int64_t orc_payload_bytes(int64_t count, int scheme, int e, int m) {
    return (count * (int64_t)orc_bit_width(scheme, e, m) + 7) / 8;
}

/* ------------------------------------------------------ codec: encode --- */
/* LSB-first bit appender: bitstream.hpp:19-59 (>32-bit fields split lo/hi is
 * transparent to the byte stream; the final byte is zero padded). */
typedef struct { uint8_t* out; int64_t pos; uint64_t acc; unsigned nb; } bitw;

static void bw_put(bitw* b, uint64_t v, unsigned w) {
    while (w > 0) {
        unsigned take = w > 32 ? 32 : w;
        uint64_t part = v & ((1ull << take) - 1);
        b->acc |= part << b->nb;
        b->nb += take;
        v = take == 64 ? 0 : v >> take;
        w -= take;
        while (b->nb >= 8) {
            b->out[b->pos++] = (uint8_t)(b->acc & 0xff);
            b->acc >>= 8;
            b->nb -= 8;
        }
    }
}

static void bw_flush(bitw* b) {
    while (b->nb > 0) {
        b->out[b->pos++] = (uint8_t)(b->acc & 0xff);
        b->acc >>= 8;
        b->nb = b->nb > 8 ? b->nb - 8 : 0;
    }
}

/* codec.cpp:103-140 compress_block; writes orc_payload_bytes() bytes */
int orc_compress_block(const double* v, int64_t n, int scheme, int e, int m, double scale,
                       uint8_t* out) {
    const unsigned width = (unsigned)orc_bit_width(scheme, e, m);
    const double inv_scale = 1.0 / scale;
    const uint64_t max_offset = (1ull << e) - 1;
    const uint64_t round_add = (m < 52) ? (1ull << (51 - m)) : 0;
    const uint64_t mant_mask = (m == 52) ? ((1ull << 52) - 1) : ((1ull << m) - 1);
    for (int64_t i = 0; i < n; ++i)
        if (!isfinite(v[i])) return ORC_INVALID_ARGUMENT;
    bitw b = {out, 0, 0, 0};
    for (int64_t i = 0; i < n; ++i) {
        double x = v[i];
        uint64_t sign = signbit(x) ? 1u : 0u;
        uint64_t field = sign << (e + m);
        if (x != 0.0) {
            const double vp = fabs(x) * inv_scale + 1.0; /* -ffp-contract=off: no FMA */
            uint64_t u = dbits(vp) + round_add;
            uint64_t offset = (u >> 52) - 1023;
            uint64_t mant = (u >> (52 - m)) & mant_mask;
            if (offset > max_offset || !isfinite(vp)) {
                offset = max_offset;
                mant = (1ull << m) - 1;
            }
            field |= (offset << m) | mant;
        }
        bw_put(&b, field, width);
    }
    bw_flush(&b);
    return ORC_OK;
}

/* codec.cpp:142-144 compress = analyze + make_descriptor(stats) + compress_block */
int orc_compress(const double* v, int64_t n, double eps, int scheme, int* e_out, int* m_out,
                 double* scale_out, uint8_t* out) {
    double mn, mx; int az;
    orc_analyze(v, n, &mn, &mx, &az);
    int e, m;
    int st = orc_make_descriptor(scheme, eps, orc_exponent_bits_for_stats(mn, mx, az), &e, &m);
    if (st) return st;
    double scale = az ? 1.0 : mn;
    st = orc_compress_block(v, n, scheme, e, m, scale, out);
    if (st) return st;
    *e_out = e; *m_out = m; *scale_out = scale;
    return ORC_OK;
}

/* ------------------------------------------------------ codec: decode --- */
/* codec.cpp:146-171 decompress_into (+ BitReader overrun -> corrupt_buffer_error,
 * bitstream.hpp:80-82) */
int orc_decompress(int scheme, int e, int m, double scale, int64_t count, const uint8_t* p,
                   int64_t len, double* out) {
    const unsigned width = (unsigned)orc_bit_width(scheme, e, m);
    if ((count * (int64_t)width + 7) / 8 > len) return ORC_CORRUPT_BUFFER;
    const uint64_t exp_mask = (1ull << e) - 1;
    const uint64_t mant_mask = (m == 52) ? ((1ull << 52) - 1) : ((1ull << m) - 1);
    int64_t pos = 0;
    uint64_t acc = 0;
    unsigned nb = 0;
    for (int64_t i = 0; i < count; ++i) {
        uint64_t field = 0;
        unsigned got = 0;
        while (got < width) { /* fields > 32 bits are read as 32 + rest, bitstream.hpp:67-74 */
            unsigned take = width - got > 32 ? 32 : width - got;
            while (nb < take) { acc |= (uint64_t)p[pos++] << nb; nb += 8; }
            field |= (acc & ((1ull << take) - 1)) << got;
            acc >>= take; nb -= take; got += take;
        }
        uint64_t sign = (field >> (e + m)) & 1u;
        uint64_t offset = (field >> m) & exp_mask;
        uint64_t mant = field & mant_mask;
        double val;
        if (offset == 0 && mant == 0) {
            val = 0.0;
        } else {
            uint64_t biased = offset + 1023 < 2046 ? offset + 1023 : 2046;
            val = (bitsd((biased << 52) | (mant << (52 - m))) - 1.0) * scale;
        }
        out[i] = sign ? -val : val;
    }
    return ORC_OK;
}

/* ------------------------------------------------------ codec: wire ----- */
/* codec.cpp:187-199 serialize: [u8 scheme][u8 e][u8 m][u8 0][f64 scale][u64 count][payload] */
int64_t orc_serialize(int scheme, int e, int m, double scale, int64_t count, const uint8_t* payload,
                      int64_t len, uint8_t* out) {
    out[0] = (uint8_t)scheme; out[1] = (uint8_t)e; out[2] = (uint8_t)m; out[3] = 0;
    memcpy(out + 4, &scale, 8);
    for (int i = 0; i < 8; ++i) out[12 + i] = (uint8_t)(((uint64_t)count >> (8 * i)) & 0xff);
    memcpy(out + 20, payload, (size_t)len);
    return 20 + len;
}

/* codec.cpp:201-225 deserialize; returns payload pointer offset via *payload_at */
int orc_deserialize(const uint8_t* data, int64_t size, int64_t* offset, int* scheme, int* e,
                    int* m, double* scale, int64_t* count, int64_t* payload_at, int64_t* len) {
    if (size < *offset || size - *offset < 20) return ORC_CORRUPT_BUFFER;
    const uint8_t* p = data + *offset;
    if (p[0] > 3) return ORC_CORRUPT_BUFFER;
    if (p[1] < 2 || p[1] > 11 || p[2] < 2 || p[2] > 52) return ORC_CORRUPT_BUFFER;
    uint64_t n = 0;
    for (int i = 0; i < 8; ++i) n |= (uint64_t)p[12 + i] << (8 * i);
    int64_t pl = (int64_t)((n * (uint64_t)orc_bit_width(p[0], p[1], p[2]) + 7) / 8);
    if (size - *offset - 20 < pl) return ORC_CORRUPT_BUFFER;
    *scheme = p[0]; *e = p[1]; *m = p[2];
    memcpy(scale, p + 4, 8);
    *count = (int64_t)n;
    *payload_at = *offset + 20;
    *len = pl;
    *offset += 20 + pl;
    return ORC_OK;
}

/* ------------------------------------------------------------- APLR ----- */
/* mixedprec.cpp:155-187 aplr_compress, from given factors (W rows x k, X cols x k,
 * column-major, sigma descending).  Column i of W is buffer i, column i of X is
 * buffer k+i.  Outputs per buffer e/m/scale and payload offsets into `blob`
 * (each payload starts at the running byte offset; offs has 2k+1 entries). */
int orc_aplr_compress(const double* W, int64_t rows, const double* X, int64_t cols, int64_t k,
                      const double* sigma, double eps, int scheme, int* e_out, int* m_out,
                      double* scale_out, int64_t* offs, uint8_t* blob) {
    offs[0] = 0;
    if (k == 0) return ORC_OK;
    const double delta = eps * sigma[0];
    const int e_w = orc_exponent_bits_for(W, rows * k);
    const int e_x = orc_exponent_bits_for(X, cols * k);
    for (int64_t i = 0; i < k; ++i) {
        double q = delta / sigma[i];
        const double eps_i = q < 0.5 ? q : 0.5; /* std::min(0.5, q) */
        for (int side = 0; side < 2; ++side) {
            const double* col = side == 0 ? W + i * rows : X + i * cols;
            int64_t len = side == 0 ? rows : cols;
            int64_t b = side == 0 ? i : k + i;
            double mn, mx; int az;
            orc_analyze(col, len, &mn, &mx, &az);
            int e, m;
            int st = orc_make_descriptor(scheme, eps_i, side == 0 ? e_w : e_x, &e, &m);
            if (st) return st;
            e_out[b] = e; m_out[b] = m; scale_out[b] = az ? 1.0 : mn;
        }
    }
    for (int64_t b = 0; b < 2 * k; ++b) {
        int64_t len = b < k ? rows : cols;
        offs[b + 1] = offs[b] + orc_payload_bytes(len, scheme, e_out[b], m_out[b]);
    }
    for (int64_t b = 0; b < 2 * k; ++b) {
        const double* col = b < k ? W + b * rows : X + (b - k) * cols;
        int64_t len = b < k ? rows : cols;
        int st = orc_compress_block(col, len, scheme, e_out[b], m_out[b], scale_out[b], blob + offs[b]);
        if (st) return st;
    }
    return ORC_OK;
}

/* ------------------------------------------ uncompressed storage ------- */
/* half.hpp:14-45 float_to_half: round to nearest even, denormals kept,
 * overflow -> inf; double_to_half = float_to_half((float)v) (half.hpp:75) */
uint16_t orc_float_to_half(float value) {
    uint32_t bits;
    memcpy(&bits, &value, 4);
    const uint32_t sign = (bits >> 16) & 0x8000u;
    const int32_t exp = (int32_t)((bits >> 23) & 0xffu) - 127 + 15;
    uint32_t mant = bits & 0x7fffffu;
    if (exp >= 31) return (uint16_t)(sign | 0x7c00u);
    if (exp <= 0) {
        if (exp < -10) return (uint16_t)sign;
        mant |= 0x800000u;
        const unsigned shift = (unsigned)(14 - exp);
        const uint32_t lsb = 1u << shift, rest = mant & (lsb - 1);
        uint32_t hm = mant >> shift;
        if (rest > (lsb >> 1) || (rest == (lsb >> 1) && (hm & 1u))) ++hm;
        return (uint16_t)(sign | hm);
    }
    uint32_t hm = mant >> 13;
    const uint32_t rest = mant & 0x1fffu;
    if (rest > 0x1000u || (rest == 0x1000u && (hm & 1u))) ++hm;
    return (uint16_t)(sign | (((uint32_t)exp << 10) + hm));
}

/* half.hpp:47-72 half_to_float */
float orc_half_to_float(uint16_t h) {
    const uint32_t sign = (uint32_t)(h & 0x8000u) << 16, exp = (h >> 10) & 0x1fu, mant = h & 0x3ffu;
    uint32_t bits;
    if (exp == 0) {
        if (mant == 0) {
            bits = sign;
        } else {
            int e = -1;
            uint32_t mm = mant;
            while (!(mm & 0x400u)) { mm <<= 1; ++e; }
            bits = sign | ((127u - 15u - (uint32_t)e) << 23) | ((mm & 0x3ffu) << 13);
        }
    } else if (exp == 31) {
        bits = sign | 0x7f800000u | (mant << 13);
    } else {
        bits = sign | ((exp - 15u + 127u) << 23) | (mant << 13);
    }
    float f;
    memcpy(&f, &bits, 4);
    return f;
}

/* mixedprec.cpp:16-41 PackedSlice::pack for n values (format 4 fp64, 5 fp32,
 * 6 fp16 in the hcmx_gpu raw-scheme numbering) */
void orc_pack_raw(const double* v, int64_t n, int fmt, uint8_t* out) {
    for (int64_t i = 0; i < n; ++i) {
        if (fmt == 4) {
            memcpy(out + 8 * i, &v[i], 8);
        } else if (fmt == 5) {
            const float f = (float)v[i];
            memcpy(out + 4 * i, &f, 4);
        } else {
            const uint16_t hv = orc_float_to_half((float)v[i]);
            memcpy(out + 2 * i, &hv, 2);
        }
    }
}

/* mixedprec.cpp:66-82 mp_partition: ranks of the FP64 / FP32 / FP16 groups */
void orc_mp_partition(const double* sigma, int64_t k, double delta, int64_t* ranks) {
    static const double rho[3] = {1.1e-16, 6.0e-8, 4.9e-4}; /* mixedprec.hpp:23 */
    ranks[0] = ranks[1] = ranks[2] = 0;
    for (int64_t j = 0; j < k; ++j) {
        const double s = sigma[j];
        if (s <= delta) continue;
        int group = 0;
        for (int i = 2; i >= 1; --i)
            if (s * rho[i] <= delta) { group = i; break; }
        ++ranks[group];
    }
}

/* ----------------------------------------------------------- matvec ----- */
/* Flattened H-matrix (the declared-only hmatrix.hpp:51-78 payload tree, leaves in
 * for_each_leaf preorder, clustering.cpp:159-166, children row-major 2i+j):
 *   leaf l: rows [row0,row1), cols [col0,col1), kind 0 = dense (one buffer,
 *   column-major scan: CodecDense hmatrix.hpp:42-44, or raw FP64), kind 1 = W
 *   Sigma X^H with one buffer per column (2k buffers: W columns then X columns,
 *   sigma[sig0 .. sig0+k): APLRLowrank mixedprec.hpp:68-82, or the MP groups of
 *   mixedprec.hpp:46-64 as raw FP64/FP32/FP16 columns), kind 2 = U V^T with one
 *   U and one V buffer (CodecLowrank hmatrix.hpp:46-49, LowrankBlock
 *   lowrank.hpp:17-29).
 *   buffer b: scheme/e/m/scale/count, payload at blob[poff[b] .. poff[b]+plen[b]);
 *   schemes 4/5/6 = uncompressed FP64/FP32/FP16 words (PackedSlice::unpack,
 *   mixedprec.cpp:43-62).
 * matvec follows hmatrix.hpp:126-128 + SPEC.md:458-466: y := alpha*M*x + beta*y
 * (beta == 0 overwrites y), alpha == 0 leaves M untouched. */
typedef struct {
    int64_t n_rows, n_cols, nleaves;
    const int64_t *row0, *row1, *col0, *col1, *kind, *rank, *buf0, *sig0;
    const double* sigma;
    const uint8_t *scheme, *e, *m;
    const double* scale;
    const int64_t *count, *poff, *plen;
    const uint8_t* blob;
    const double* raw;
} orc_hmat;

typedef struct {
    const orc_hmat* h;
    const double* x;
    double* z; /* private accumulator n_rows (n_cols when transposed) */
    int64_t l0, l1;
    int status;
    int transpose; /* hmatrix.hpp:128: y := alpha M^T x + beta y */
} mv_job;

static int decode_buf(const orc_hmat* h, int64_t b, double* out) {
    const int sc = h->scheme[b];
    if (sc >= 4) { /* uncompressed words */
        const uint8_t* p = h->blob + h->poff[b];
        const int64_t n = h->count[b], esz = sc == 4 ? 8 : sc == 5 ? 4 : 2;
        if (sc > 6 || n * esz > h->plen[b]) return ORC_CORRUPT_BUFFER;
        for (int64_t i = 0; i < n; ++i) {
            if (sc == 4) {
                memcpy(&out[i], p + 8 * i, 8);
            } else if (sc == 5) {
                float f;
                memcpy(&f, p + 4 * i, 4);
                out[i] = (double)f;
            } else {
                uint16_t hv;
                memcpy(&hv, p + 2 * i, 2);
                out[i] = (double)orc_half_to_float(hv);
            }
        }
        return ORC_OK;
    }
    return orc_decompress(sc, h->e[b], h->m[b], h->scale[b], h->count[b], h->blob + h->poff[b], h->plen[b],
                          out);
}

static void* mv_worker(void* arg) {
    mv_job* j = (mv_job*)arg;
    const orc_hmat* h = j->h;
    int64_t maxe = 0;
    for (int64_t l = j->l0; l < j->l1; ++l) {
        int64_t r = h->row1[l] - h->row0[l], c = h->col1[l] - h->col0[l];
        int64_t need = h->kind[l] != 0 ? (r + c) * h->rank[l] + h->rank[l] : r * c;
        if (need > maxe) maxe = need;
    }
    double* tmp = (double*)malloc(sizeof(double) * (size_t)(maxe + 1));
    for (int64_t l = j->l0; l < j->l1 && j->status == 0; ++l) {
        const int64_t r0 = h->row0[l], c0 = h->col0[l];
        const int64_t rows = h->row1[l] - r0, cols = h->col1[l] - c0;
        if (h->kind[l] == 0) {
            if (h->count[h->buf0[l]] != rows * cols) { j->status = ORC_INVALID_ARGUMENT; break; }
            j->status = decode_buf(h, h->buf0[l], tmp);
            const double* A = tmp;
            if (j->transpose) {
                for (int64_t cc = 0; cc < cols; ++cc) {
                    const double* a = A + cc * rows;
                    double s = 0.0;
                    for (int64_t rr = 0; rr < rows; ++rr) s += a[rr] * j->x[r0 + rr];
                    j->z[c0 + cc] += s;
                }
            } else {
                for (int64_t cc = 0; cc < cols; ++cc) {
                    const double xv = j->x[c0 + cc];
                    const double* a = A + cc * rows;
                    for (int64_t rr = 0; rr < rows; ++rr) j->z[r0 + rr] += a[rr] * xv;
                }
            }
        } else {
            const int64_t k = h->rank[l];
            double* Wd = tmp;
            double* Xd = tmp + rows * k;
            double* t = Xd + cols * k;
            if (h->kind[l] == 2) { /* one U and one V buffer, column-major */
                if (k > 0) {
                    j->status |= decode_buf(h, h->buf0[l], Wd);
                    j->status |= decode_buf(h, h->buf0[l] + 1, Xd);
                }
            } else {
                for (int64_t i = 0; i < k && j->status == 0; ++i) {
                    j->status |= decode_buf(h, h->buf0[l] + i, Wd + i * rows);
                    j->status |= decode_buf(h, h->buf0[l] + k + i, Xd + i * cols);
                }
            }
            /* mixedprec.cpp:203-208: U = W diag(sigma), V = X; y_t += U (V^T x_s)
             * (sigma = 1 for U V^T leaves); transposed: y_s += V (U^T x_t) */
            const double* in = j->transpose ? Wd : Xd;
            const double* outf = j->transpose ? Xd : Wd;
            const int64_t nin = j->transpose ? rows : cols, nout = j->transpose ? cols : rows;
            const int64_t oin = j->transpose ? r0 : c0, oout = j->transpose ? c0 : r0;
            for (int64_t i = 0; i < k; ++i) {
                double s = 0.0;
                const double* xc = in + i * nin;
                for (int64_t cc = 0; cc < nin; ++cc) s += xc[cc] * j->x[oin + cc];
                t[i] = h->kind[l] == 2 ? s : s * h->sigma[h->sig0[l] + i];
            }
            for (int64_t i = 0; i < k; ++i) {
                const double* wc = outf + i * nout;
                for (int64_t rr = 0; rr < nout; ++rr) j->z[oout + rr] += wc[rr] * t[i];
            }
        }
    }
    free(tmp);
    return NULL;
}

/* leaf ranges split by cumulative value count so threads get even work; the
 * private accumulators are summed in thread order (deterministic for fixed T). */
int orc_hmat_matvec_t(const orc_hmat* h, double alpha, const double* x, double beta, double* y,
                      int threads, int transpose) {
    if (threads < 1) threads = 1;
    const int64_t ny = transpose ? h->n_cols : h->n_rows;
    for (int64_t i = 0; i < ny; ++i) y[i] = beta == 0.0 ? 0.0 : beta * y[i];
    if (alpha == 0.0) return ORC_OK;
    double* work = (double*)malloc(sizeof(double) * (size_t)h->nleaves + 8);
    double total = 0.0;
    for (int64_t l = 0; l < h->nleaves; ++l) {
        double r = (double)(h->row1[l] - h->row0[l]), c = (double)(h->col1[l] - h->col0[l]);
        work[l] = h->kind[l] != 0 ? (r + c) * (double)h->rank[l] : r * c;
        total += work[l];
    }
    mv_job* jobs = (mv_job*)calloc((size_t)threads, sizeof(mv_job));
    pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    int64_t l = 0;
    double acc = 0.0;
    for (int t = 0; t < threads; ++t) {
        jobs[t].h = h; jobs[t].x = x; jobs[t].l0 = l; jobs[t].transpose = transpose;
        double target = total * (double)(t + 1) / (double)threads;
        while (l < h->nleaves && (t == threads - 1 || acc + work[l] * 0.5 <= target)) acc += work[l++];
        jobs[t].l1 = l;
        jobs[t].z = (double*)calloc((size_t)ny, sizeof(double));
    }
    for (int t = 1; t < threads; ++t) pthread_create(&tid[t], NULL, mv_worker, &jobs[t]);
    mv_worker(&jobs[0]);
    for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
    int st = ORC_OK;
    for (int t = 0; t < threads; ++t) {
        if (jobs[t].status) st = jobs[t].status;
        for (int64_t i = 0; i < ny; ++i) y[i] += alpha * jobs[t].z[i];
        free(jobs[t].z);
    }
    free(jobs); free(tid); free(work);
    return st;
}

int orc_hmat_matvec(const orc_hmat* h, double alpha, const double* x, double beta, double* y,
                    int threads) {
    return orc_hmat_matvec_t(h, alpha, x, beta, y, threads, 0);
}

/* flat-argument wrapper for ctypes */
int orc_hmat_matvec_flat(int64_t n_rows, int64_t n_cols, int64_t nleaves, const int64_t* row0,
                         const int64_t* row1, const int64_t* col0, const int64_t* col1,
                         const int64_t* kind, const int64_t* rank, const int64_t* buf0,
                         const int64_t* sig0, const double* sigma, const uint8_t* scheme,
                         const uint8_t* e, const uint8_t* m, const double* scale,
                         const int64_t* count, const int64_t* poff, const int64_t* plen,
                         const uint8_t* blob, const double* raw, double alpha, const double* x,
                         double beta, double* y, int threads) {
    orc_hmat h = {n_rows, n_cols, nleaves, row0, row1, col0, col1, kind, rank, buf0, sig0,
                  sigma, scheme, e, m, scale, count, poff, plen, blob, raw};
    return orc_hmat_matvec(&h, alpha, x, beta, y, threads);
}

/* transpose = 1: y (n_cols) := alpha M^T x + beta y (hmatrix.hpp:128) */
int orc_hmat_matvec_t_flat(int64_t n_rows, int64_t n_cols, int64_t nleaves, const int64_t* row0,
                           const int64_t* row1, const int64_t* col0, const int64_t* col1,
                           const int64_t* kind, const int64_t* rank, const int64_t* buf0,
                           const int64_t* sig0, const double* sigma, const uint8_t* scheme,
                           const uint8_t* e, const uint8_t* m, const double* scale,
                           const int64_t* count, const int64_t* poff, const int64_t* plen,
                           const uint8_t* blob, const double* raw, double alpha, const double* x,
                           double beta, double* y, int threads, int transpose) {
    orc_hmat h = {n_rows, n_cols, nleaves, row0, row1, col0, col1, kind, rank, buf0, sig0,
                  sigma, scheme, e, m, scale, count, poff, plen, blob, raw};
    return orc_hmat_matvec_t(&h, alpha, x, beta, y, threads, transpose);
}

/* ------------------------------------------------- batched codec (CPU) --- */
/* Batched compress of independent buffers over T threads (the CPU baseline
 * harness; the reference functions are pure). */
typedef struct {
    const double* v; const int64_t* voff; const int64_t* cnt; double eps; int scheme;
    int* e; int* m; double* scale; const int64_t* poff; uint8_t* blob;
    const int64_t* plen_out_unused; int64_t b0, b1; int status; int mode;
    const uint8_t* cblob; double* dout;
} cb_job;

static void* cb_worker(void* arg) {
    cb_job* j = (cb_job*)arg;
    for (int64_t b = j->b0; b < j->b1; ++b) {
        int st;
        if (j->mode == 0)
            st = orc_compress(j->v + j->voff[b], j->cnt[b], j->eps, j->scheme, &j->e[b], &j->m[b],
                              &j->scale[b], j->blob + j->poff[b]);
        else
            st = orc_decompress(j->scheme, j->e[b], j->m[b], j->scale[b], j->cnt[b],
                                j->cblob + j->poff[b], 1ll << 62, j->dout + j->voff[b]);
        if (st) j->status = st;
    }
    return NULL;
}

static int run_batch(cb_job* proto, int64_t nbuf, int threads) {
    if (threads < 1) threads = 1;
    cb_job* jobs = (cb_job*)calloc((size_t)threads, sizeof(cb_job));
    pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    for (int t = 0; t < threads; ++t) {
        jobs[t] = *proto;
        jobs[t].b0 = nbuf * t / threads;
        jobs[t].b1 = nbuf * (t + 1) / threads;
    }
    for (int t = 1; t < threads; ++t) pthread_create(&tid[t], NULL, cb_worker, &jobs[t]);
    cb_worker(&jobs[0]);
    for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
    int st = 0;
    for (int t = 0; t < threads; ++t) if (jobs[t].status) st = jobs[t].status;
    free(jobs); free(tid);
    return st;
}

/* payload slot b starts at poff[b] (caller sized slots for the worst case 8*cnt) */
int orc_compress_batch(const double* v, const int64_t* voff, const int64_t* cnt, int64_t nbuf,
                       double eps, int scheme, int* e, int* m, double* scale, const int64_t* poff,
                       uint8_t* blob, int threads) {
    cb_job p; memset(&p, 0, sizeof p);
    p.v = v; p.voff = voff; p.cnt = cnt; p.eps = eps; p.scheme = scheme; p.e = e; p.m = m;
    p.scale = scale; p.poff = poff; p.blob = blob; p.mode = 0;
    return run_batch(&p, nbuf, threads);
}

int orc_decompress_batch(const uint8_t* blob, const int64_t* poff, const int64_t* cnt,
                         const int64_t* voff, int64_t nbuf, int scheme, int* e, int* m,
                         double* scale, double* out, int threads) {
    cb_job p; memset(&p, 0, sizeof p);
    p.cblob = blob; p.poff = poff; p.cnt = cnt; p.voff = voff; p.scheme = scheme; p.e = e;
    p.m = m; p.scale = scale; p.dout = out; p.mode = 1;
    return run_batch(&p, nbuf, threads);
}
