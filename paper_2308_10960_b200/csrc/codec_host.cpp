// codec_host.cpp -- the codec's per-buffer layout rules on the host, plus the
// host-pointer and wire-format entry points of the C-ABI.
//
// The layout rules are scalar work per buffer (a handful of flops per 4096
// values), so they stay on the host where glibc's log2 gives exactly the
// reference's decisions (SURVEY 7 "Descriptor selection": CUDA's double log2
// is only <= 1 ulp, which could flip e next to the 2^k - 2 thresholds).  The
// device computes the per-buffer min/max (exact comparisons) that feed them.
//
// Compiled with g++ -ffp-contract=off (paper_2308_10960_b200/build.py).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>

#include "internal.h"

namespace hcmx_gpu {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& s) { g_last_error = s; }

// codec.hpp:40-49
unsigned alignment_unit(int scheme) {
    switch (scheme) {
        case HCMX_AFL: return 1;
        case HCMX_AFLP:
        case HCMX_BFL: return 8;
        case HCMX_DFL: return 16;
    }
    throw invalid_argument("unknown codec scheme");
}

// codec.hpp:51-55
unsigned bit_width(int scheme, unsigned e, unsigned m) {
    const unsigned unit = alignment_unit(scheme);
    const unsigned w = 1u + e + m;
    return w + (unit - w % unit) % unit;
}

// codec.cpp:62-67: m = clamp(ceil(-log2 eps) - 1, 2, 52)
uint8_t mantissa_bits_for(double eps) {
    if (!(eps > 0.0) || !(eps < 1.0))
        throw invalid_argument("mantissa_bits_for: eps must lie in (0, 1)");
    const double bits = std::ceil(-std::log2(eps)) - 1.0;
    return static_cast<uint8_t>(std::clamp(bits, 2.0, 52.0));
}

// codec.cpp:69-75: e = clamp(ceil(log2(log2 max - log2 min + 2)), 2, 11)
uint8_t exponent_bits_for(const hcmx_stats& st) {
    if (st.all_zero) return 2;
    const double span = std::log2(st.max_mag) - std::log2(st.min_mag) + 1.0;
    const double bits = std::ceil(std::log2(span + 1.0));
    return static_cast<uint8_t>(std::clamp(bits, 2.0, 11.0));
}

// codec.cpp:25-30 (non-AFL schemes widen m to fill the 8/8/16-bit unit, cap 52)
static uint8_t align_mantissa(int scheme, unsigned e, unsigned m) {
    const unsigned unit = alignment_unit(scheme);
    unsigned w = 1u + e + m;
    w += (unit - w % unit) % unit;
    return static_cast<uint8_t>(std::min(52u, w - 1u - e));
}

// codec.cpp:86-101
hcmx_descriptor make_descriptor(int scheme, double eps, double scale, uint8_t exp_bits) {
    hcmx_descriptor d{};
    d.scheme = static_cast<uint8_t>(scheme);
    d.scale = scale;
    switch (scheme) {
        case HCMX_AFL:
        case HCMX_AFLP: d.exp_bits = exp_bits; break;
        case HCMX_BFL: d.exp_bits = 8; break;
        case HCMX_DFL: d.exp_bits = 11; break;
        default: throw invalid_argument("unknown codec scheme");
    }
    d.mant_bits = mantissa_bits_for(eps);
    if (scheme != HCMX_AFL) d.mant_bits = align_mantissa(scheme, d.exp_bits, d.mant_bits);
    d.bit_width = static_cast<uint8_t>(bit_width(scheme, d.exp_bits, d.mant_bits));
    return d;
}

// codec.cpp:81-84
hcmx_descriptor make_descriptor(int scheme, double eps, const hcmx_stats& st) {
    return make_descriptor(scheme, eps, st.all_zero ? 1.0 : st.min_mag, exponent_bits_for(st));
}

}  // namespace hcmx_gpu

using namespace hcmx_gpu;

extern "C" {

const char* hcmx_gpu_last_error(void) { return g_last_error.c_str(); }

int hcmx_gpu_version(void) { return 1; }

int hcmx_gpu_mantissa_bits_for(double eps, uint8_t* out) {
    return guarded([&] { *out = mantissa_bits_for(eps); });
}

int hcmx_gpu_exponent_bits_for(const hcmx_stats* st, uint8_t* out) {
    return guarded([&] { *out = exponent_bits_for(*st); });
}

int hcmx_gpu_make_descriptor(int scheme, double eps, const hcmx_stats* st, hcmx_descriptor* out) {
    return guarded([&] { *out = make_descriptor(scheme, eps, *st); });
}

int hcmx_gpu_make_descriptor_pinned(int scheme, double eps, double scale, uint8_t exp_bits,
                                    hcmx_descriptor* out) {
    return guarded([&] { *out = make_descriptor(scheme, eps, scale, exp_bits); });
}

unsigned hcmx_gpu_bit_width(const hcmx_descriptor* d) {
    return bit_width(d->scheme, d->exp_bits, d->mant_bits);
}

uint64_t hcmx_gpu_payload_bytes(uint64_t count, const hcmx_descriptor* d) {
    return payload_bytes(count, bit_width(d->scheme, d->exp_bits, d->mant_bits));
}

uint64_t hcmx_gpu_compressed_size(uint64_t count, const hcmx_descriptor* d) {
    return 20 + hcmx_gpu_payload_bytes(count, d);
}

// codec.cpp:187-199
uint64_t hcmx_gpu_serialize(const hcmx_descriptor* d, uint64_t count, const uint8_t* payload,
                            uint64_t len, uint8_t* out) {
    out[0] = d->scheme;
    out[1] = d->exp_bits;
    out[2] = d->mant_bits;
    out[3] = 0;
    std::memcpy(out + 4, &d->scale, 8);
    for (int i = 0; i < 8; ++i) out[12 + i] = static_cast<uint8_t>((count >> (8 * i)) & 0xffu);
    if (len) std::memcpy(out + 20, payload, len);
    return 20 + len;
}

// codec.cpp:201-225
int hcmx_gpu_deserialize(const uint8_t* data, uint64_t size, uint64_t* offset,
                         hcmx_descriptor* d, uint64_t* count, uint64_t* payload_at,
                         uint64_t* payload_len) {
    return guarded([&] {
        if (size < *offset || size - *offset < 20)
            throw corrupt_buffer("deserialize: truncated header");
        const uint8_t* p = data + *offset;
        if (p[0] > 3) throw corrupt_buffer("deserialize: unknown scheme tag");
        if (p[1] < 2 || p[1] > 11 || p[2] < 2 || p[2] > 52)
            throw corrupt_buffer("deserialize: invalid bit widths");
        hcmx_descriptor r{};
        r.scheme = p[0];
        r.exp_bits = p[1];
        r.mant_bits = p[2];
        r.bit_width = static_cast<uint8_t>(bit_width(r.scheme, r.exp_bits, r.mant_bits));
        std::memcpy(&r.scale, p + 4, 8);
        uint64_t n = 0;
        for (int i = 0; i < 8; ++i) n |= static_cast<uint64_t>(p[12 + i]) << (8 * i);
        const uint64_t len = payload_bytes(n, r.bit_width);
        if (size - *offset - 20 < len) throw corrupt_buffer("deserialize: truncated payload");
        *d = r;
        *count = n;
        *payload_at = *offset + 20;
        *payload_len = len;
        *offset += 20 + len;
    });
}

}  // extern "C"
