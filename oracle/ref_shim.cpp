// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrappers around the UNMODIFIED reference codec, compiled from
// /root/reference/proj/src/codec.cpp where it lies (oracle/Makefile; output in
// the git-ignored oracle/_ref/).  No reference source is copied into this repo.
//
// What is reference code and what is restated here:
//   * codec::analyze / mantissa_bits_for / exponent_bits_for / make_descriptor /
//     compress / compress_block / decompress_into / serialize / deserialize /
//     compressed_size  -> the reference itself (codec.cpp:44-225).
//   * APLR glue -> restated from mixedprec.cpp:155-187 (mixedprec.cpp needs
//     Eigen, which is absent), calling only the reference codec functions.
//   * H-matvec  -> restated from hmatrix.hpp:126-128 + SPEC.md:458-466 (the
//     reference declares matvec but ships no implementation), decoding every
//     leaf with the reference decompress_into.
//   * batch drivers -> thread fan-out over independent buffers (SPEC.md:327-328:
//     the codec functions are pure).
// Used by tests/ as the parity pin and by bench.py --impl reference.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <random>
#include <span>
#include <stdexcept>
#include <thread>
#include <vector>

#include "hcmx/codec.hpp"
#include "hcmx/half.hpp"

using namespace hcmx;
using codec::Scheme;

namespace {

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (const corrupt_buffer_error&) {
        return 2;
    } catch (...) {
        return 3;
    }
}

codec::CompressedBuffer make_buf(int scheme, int e, int m, double scale, std::int64_t count,
                                 const std::uint8_t* p, std::int64_t len) {
    codec::CompressedBuffer b;
    b.descriptor.scheme = static_cast<Scheme>(scheme);
    b.descriptor.exp_bits = static_cast<std::uint8_t>(e);
    b.descriptor.mant_bits = static_cast<std::uint8_t>(m);
    b.descriptor.scale = scale;
    b.count = static_cast<std::uint64_t>(count);
    b.payload.assign(p, p + len);
    return b;
}

template <class F>
int fan_out(std::int64_t n, int threads, F&& body) {
    threads = std::max(1, threads);
    std::vector<int> st(threads, 0);
    std::vector<std::thread> pool;
    auto run = [&](int t) {
        const std::int64_t b0 = n * t / threads, b1 = n * (t + 1) / threads;
        for (std::int64_t b = b0; b < b1; ++b) {
            int s = guarded([&] { body(b); });
            if (s) st[t] = s;
        }
    };
    for (int t = 1; t < threads; ++t) pool.emplace_back(run, t);
    run(0);
    for (auto& th : pool) th.join();
    for (int s : st)
        if (s) return s;
    return 0;
}

} // namespace

extern "C" {

// half.hpp conversions, header-only reference code (pins the restatement)
std::uint16_t ref_float_to_half(float v) { return hcmx::mp::float_to_half(v); }
float ref_half_to_float(std::uint16_t h) { return hcmx::mp::half_to_float(h); }

void ref_mt64_raw(std::uint64_t seed, std::int64_t n, std::uint64_t* out) {
    std::mt19937_64 g(seed);
    for (std::int64_t i = 0; i < n; ++i) out[i] = g();
}

void ref_analyze(const double* v, std::int64_t n, double* mn, double* mx, int* az) {
    auto st = codec::analyze(std::span<const double>(v, static_cast<std::size_t>(n)));
    *mn = st.min_mag;
    *mx = st.max_mag;
    *az = st.all_zero ? 1 : 0;
}

int ref_mantissa_bits_for(double eps, int* out) {
    return guarded([&] { *out = codec::mantissa_bits_for(eps); });
}

int ref_exponent_bits_for(const double* v, std::int64_t n) {
    return codec::exponent_bits_for(std::span<const double>(v, static_cast<std::size_t>(n)));
}

int ref_exponent_bits_for_stats(double mn, double mx, int az) {
    codec::BlockStats st{mn, mx, az != 0};
    return codec::exponent_bits_for(st);
}

int ref_make_descriptor_stats(int scheme, double eps, double mn, double mx, int az, int* e, int* m,
                              double* scale) {
    return guarded([&] {
        auto d = codec::make_descriptor(static_cast<Scheme>(scheme), eps,
                                        codec::BlockStats{mn, mx, az != 0});
        *e = d.exp_bits;
        *m = d.mant_bits;
        *scale = d.scale;
    });
}

int ref_make_descriptor(int scheme, double eps, double scale, int exp_bits, int* e, int* m) {
    return guarded([&] {
        auto d = codec::make_descriptor(static_cast<Scheme>(scheme), eps, scale,
                                        static_cast<std::uint8_t>(exp_bits));
        *e = d.exp_bits;
        *m = d.mant_bits;
    });
}

int ref_bit_width(int scheme, int e, int m) {
    codec::FormatDescriptor d;
    d.scheme = static_cast<Scheme>(scheme);
    d.exp_bits = static_cast<std::uint8_t>(e);
    d.mant_bits = static_cast<std::uint8_t>(m);
    return static_cast<int>(d.bit_width());
}

std::int64_t ref_compressed_size(std::int64_t count, int scheme, int e, int m) {
    codec::FormatDescriptor d;
    d.scheme = static_cast<Scheme>(scheme);
    d.exp_bits = static_cast<std::uint8_t>(e);
    d.mant_bits = static_cast<std::uint8_t>(m);
    return static_cast<std::int64_t>(codec::compressed_size(static_cast<std::uint64_t>(count), d));
}

// out must hold cap bytes; *len receives the payload length
int ref_compress(const double* v, std::int64_t n, double eps, int scheme, int* e, int* m,
                 double* scale, std::uint8_t* out, std::int64_t cap, std::int64_t* len) {
    return guarded([&] {
        auto b = codec::compress(std::span<const double>(v, static_cast<std::size_t>(n)), eps,
                                 static_cast<Scheme>(scheme));
        if (static_cast<std::int64_t>(b.payload.size()) > cap)
            throw std::runtime_error("cap");
        std::memcpy(out, b.payload.data(), b.payload.size());
        *len = static_cast<std::int64_t>(b.payload.size());
        *e = b.descriptor.exp_bits;
        *m = b.descriptor.mant_bits;
        *scale = b.descriptor.scale;
    });
}

int ref_compress_block(const double* v, std::int64_t n, int scheme, int e, int m, double scale,
                       std::uint8_t* out, std::int64_t cap, std::int64_t* len) {
    return guarded([&] {
        codec::FormatDescriptor d;
        d.scheme = static_cast<Scheme>(scheme);
        d.exp_bits = static_cast<std::uint8_t>(e);
        d.mant_bits = static_cast<std::uint8_t>(m);
        d.scale = scale;
        auto b = codec::compress_block(std::span<const double>(v, static_cast<std::size_t>(n)), d);
        if (static_cast<std::int64_t>(b.payload.size()) > cap)
            throw std::runtime_error("cap");
        std::memcpy(out, b.payload.data(), b.payload.size());
        *len = static_cast<std::int64_t>(b.payload.size());
    });
}

int ref_decompress(int scheme, int e, int m, double scale, std::int64_t count,
                   const std::uint8_t* p, std::int64_t len, double* out) {
    return guarded([&] { codec::decompress_into(make_buf(scheme, e, m, scale, count, p, len), out); });
}

std::int64_t ref_serialize(int scheme, int e, int m, double scale, std::int64_t count,
                           const std::uint8_t* p, std::int64_t len, std::uint8_t* out) {
    std::vector<std::uint8_t> bytes;
    codec::serialize(make_buf(scheme, e, m, scale, count, p, len), bytes);
    std::memcpy(out, bytes.data(), bytes.size());
    return static_cast<std::int64_t>(bytes.size());
}

int ref_deserialize(const std::uint8_t* data, std::int64_t size, std::int64_t* offset, int* scheme,
                    int* e, int* m, double* scale, std::int64_t* count, std::int64_t* payload_at,
                    std::int64_t* len) {
    return guarded([&] {
        std::size_t off = static_cast<std::size_t>(*offset);
        auto b = codec::deserialize(data, static_cast<std::size_t>(size), off);
        *scheme = static_cast<int>(b.descriptor.scheme);
        *e = b.descriptor.exp_bits;
        *m = b.descriptor.mant_bits;
        *scale = b.descriptor.scale;
        *count = static_cast<std::int64_t>(b.count);
        *payload_at = static_cast<std::int64_t>(off - b.payload.size());
        *len = static_cast<std::int64_t>(b.payload.size());
        *offset = static_cast<std::int64_t>(off);
    });
}

// Batched compress: buffer b = v[voff[b] .. voff[b]+cnt[b]), payload written at
// blob + poff[b] (slots sized by the caller), length into plen[b].
int ref_compress_batch(const double* v, const std::int64_t* voff, const std::int64_t* cnt,
                       std::int64_t nbuf, double eps, int scheme, int* e, int* m, double* scale,
                       const std::int64_t* poff, std::uint8_t* blob, std::int64_t* plen,
                       int threads) {
    return fan_out(nbuf, threads, [&](std::int64_t b) {
        auto r = codec::compress(
            std::span<const double>(v + voff[b], static_cast<std::size_t>(cnt[b])), eps,
            static_cast<Scheme>(scheme));
        std::memcpy(blob + poff[b], r.payload.data(), r.payload.size());
        plen[b] = static_cast<std::int64_t>(r.payload.size());
        e[b] = r.descriptor.exp_bits;
        m[b] = r.descriptor.mant_bits;
        scale[b] = r.descriptor.scale;
    });
}

int ref_decompress_batch(const std::uint8_t* blob, const std::int64_t* poff,
                         const std::int64_t* plen, const std::int64_t* cnt,
                         const std::int64_t* voff, std::int64_t nbuf, int scheme, const int* e,
                         const int* m, const double* scale, double* out, int threads) {
    return fan_out(nbuf, threads, [&](std::int64_t b) {
        codec::decompress_into(
            make_buf(scheme, e[b], m[b], scale[b], cnt[b], blob + poff[b], plen[b]),
            out + voff[b]);
    });
}

// APLR glue restated from mixedprec.cpp:155-187 on given factors (the SVD that
// produces W, sigma, X needs Eigen and is not reproducible here).
// Buffers: W column i -> i, X column i -> k+i; payload b at blob + offs[b].
int ref_aplr_compress(const double* W, std::int64_t rows, const double* X, std::int64_t cols,
                      std::int64_t k, const double* sigma, double eps, int scheme, int* e_out,
                      int* m_out, double* scale_out, std::int64_t* offs, std::uint8_t* blob) {
    return guarded([&] {
        offs[0] = 0;
        if (k == 0)
            return;
        const double delta = eps * sigma[0];
        const auto e_w = codec::exponent_bits_for(
            std::span<const double>(W, static_cast<std::size_t>(rows * k)));
        const auto e_x = codec::exponent_bits_for(
            std::span<const double>(X, static_cast<std::size_t>(cols * k)));
        std::vector<codec::CompressedBuffer> bufs;
        for (std::int64_t i = 0; i < k; ++i) {
            const double eps_i = std::min(0.5, delta / sigma[i]);
            const std::span<const double> wc(W + i * rows, static_cast<std::size_t>(rows));
            const auto ws = codec::analyze(wc);
            bufs.push_back(codec::compress_block(
                wc, codec::make_descriptor(static_cast<Scheme>(scheme), eps_i,
                                           ws.all_zero ? 1.0 : ws.min_mag, e_w)));
        }
        for (std::int64_t i = 0; i < k; ++i) {
            const double eps_i = std::min(0.5, delta / sigma[i]);
            const std::span<const double> xc(X + i * cols, static_cast<std::size_t>(cols));
            const auto xs = codec::analyze(xc);
            bufs.push_back(codec::compress_block(
                xc, codec::make_descriptor(static_cast<Scheme>(scheme), eps_i,
                                           xs.all_zero ? 1.0 : xs.min_mag, e_x)));
        }
        for (std::int64_t b = 0; b < 2 * k; ++b) {
            e_out[b] = bufs[b].descriptor.exp_bits;
            m_out[b] = bufs[b].descriptor.mant_bits;
            scale_out[b] = bufs[b].descriptor.scale;
            std::memcpy(blob + offs[b], bufs[b].payload.data(), bufs[b].payload.size());
            offs[b + 1] = offs[b] + static_cast<std::int64_t>(bufs[b].payload.size());
        }
    });
}

// H-matvec restated (hmatrix.hpp:126-128) over the flattened
// leaf list (see oracle/hcmx_oracle.c for the layout), decoding with the
// reference decompress_into.  Threads take contiguous leaf ranges balanced by
// value count and accumulate privately; partial vectors are summed in thread
// order, so the result is deterministic for a fixed thread count.
int ref_hmat_matvec_flat(std::int64_t n_rows, std::int64_t /*n_cols*/, std::int64_t nleaves,
                         const std::int64_t* row0, const std::int64_t* row1,
                         const std::int64_t* col0, const std::int64_t* col1,
                         const std::int64_t* kind, const std::int64_t* rank,
                         const std::int64_t* buf0, const std::int64_t* sig0, const double* sigma,
                         const std::uint8_t* scheme, const std::uint8_t* e, const std::uint8_t* m,
                         const double* scale, const std::int64_t* count, const std::int64_t* poff,
                         const std::int64_t* plen, const std::uint8_t* blob, const double* raw,
                         double alpha, const double* x, double beta, double* y, int threads) {
    return guarded([&] {
        for (std::int64_t i = 0; i < n_rows; ++i)
            y[i] = beta == 0.0 ? 0.0 : beta * y[i];
        if (alpha == 0.0)
            return;
        threads = std::max(1, threads);
        std::vector<double> work(nleaves);
        double total = 0;
        for (std::int64_t l = 0; l < nleaves; ++l) {
            const double r = double(row1[l] - row0[l]), c = double(col1[l] - col0[l]);
            work[l] = kind[l] == 1 ? (r + c) * double(rank[l]) : r * c;
            total += work[l];
        }
        std::vector<std::int64_t> cut(threads + 1, nleaves);
        cut[0] = 0;
        {
            std::int64_t l = 0;
            double acc = 0;
            for (int t = 0; t < threads - 1; ++t) {
                const double target = total * double(t + 1) / double(threads);
                while (l < nleaves && acc + work[l] * 0.5 <= target) acc += work[l++];
                cut[t + 1] = l;
            }
        }
        auto buf = [&](std::int64_t b) {
            return make_buf(scheme[b], e[b], m[b], scale[b], count[b], blob + poff[b], plen[b]);
        };
        std::vector<std::vector<double>> z(threads, std::vector<double>(n_rows, 0.0));
        std::vector<int> st(threads, 0);
        auto run = [&](int t) {
            st[t] = guarded([&] {
                std::vector<double> tmp, wd, xd, tv;
                for (std::int64_t l = cut[t]; l < cut[t + 1]; ++l) {
                    const std::int64_t r0 = row0[l], c0 = col0[l];
                    const std::int64_t rows = row1[l] - r0, cols = col1[l] - c0;
                    if (kind[l] != 1) {
                        const double* A;
                        if (kind[l] == 0) {
                            tmp.resize(rows * cols);
                            codec::decompress_into(buf(buf0[l]), tmp.data());
                            A = tmp.data();
                        } else {
                            A = raw + buf0[l];
                        }
                        for (std::int64_t cc = 0; cc < cols; ++cc) {
                            const double xv = x[c0 + cc];
                            for (std::int64_t rr = 0; rr < rows; ++rr)
                                z[t][r0 + rr] += A[cc * rows + rr] * xv;
                        }
                    } else {
                        const std::int64_t k = rank[l];
                        wd.resize(rows * k);
                        xd.resize(cols * k);
                        tv.resize(k);
                        for (std::int64_t i = 0; i < k; ++i) {
                            codec::decompress_into(buf(buf0[l] + i), wd.data() + i * rows);
                            codec::decompress_into(buf(buf0[l] + k + i), xd.data() + i * cols);
                        }
                        for (std::int64_t i = 0; i < k; ++i) {
                            double s = 0;
                            for (std::int64_t cc = 0; cc < cols; ++cc)
                                s += xd[i * cols + cc] * x[c0 + cc];
                            tv[i] = s * sigma[sig0[l] + i];
                        }
                        for (std::int64_t i = 0; i < k; ++i)
                            for (std::int64_t rr = 0; rr < rows; ++rr)
                                z[t][r0 + rr] += wd[i * rows + rr] * tv[i];
                    }
                }
            });
        };
        std::vector<std::thread> pool;
        for (int t = 1; t < threads; ++t) pool.emplace_back(run, t);
        run(0);
        for (auto& th : pool) th.join();
        for (int t = 0; t < threads; ++t) {
            if (st[t] == 1) throw std::invalid_argument("matvec");
            if (st[t] == 2) throw corrupt_buffer_error("matvec");
            if (st[t]) throw std::runtime_error("matvec");
            for (std::int64_t i = 0; i < n_rows; ++i) y[i] += alpha * z[t][i];
        }
    });
}

} // extern "C"
