// hcmx_gpu.hpp -- header-only C++20 shim over the C-ABI (hcmx_gpu.h) that keeps
// the reference's API surface (proj/include/hcmx/codec.hpp:16-110 and the
// matvec of hmatrix.hpp:126-128) so a caller of the reference can switch with a
// namespace alias:
//
//     #include <hcmx_gpu.hpp>
//     namespace codec = hcmx_gpu::codec;          // instead of hcmx::codec
//
// Statuses map back to the reference's exception types: HCMX_INVALID_ARGUMENT
// -> std::invalid_argument, HCMX_CORRUPT_BUFFER -> hcmx::corrupt_buffer_error
// (common.hpp:17-19: the reference's own type when its headers are on the
// include path, else an identical declaration), anything else ->
// std::runtime_error.  Where Eigen is available the hmatrix.hpp:126-128
// signature matvec(double, const M&, const Eigen::VectorXd&, double,
// Eigen::VectorXd&, bool) is provided too.
#ifndef HCMX_GPU_HPP
#define HCMX_GPU_HPP

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "hcmx_gpu.h"

#if __has_include(<hcmx/common.hpp>)
#include <hcmx/common.hpp>  // the reference's hcmx::corrupt_buffer_error
#else
namespace hcmx {
// proj/include/hcmx/common.hpp:17-19 (same name, base and constructor)
class corrupt_buffer_error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
}  // namespace hcmx
#endif

#if __has_include(<Eigen/Dense>)
#include <Eigen/Dense>
#define HCMX_GPU_HAVE_EIGEN 1
#endif

namespace hcmx_gpu {

// a reference caller's `catch (const hcmx::corrupt_buffer_error&)` catches it
using corrupt_buffer_error = hcmx::corrupt_buffer_error;

inline void check(int status, const char* what) {
    if (status == HCMX_OK) return;
    const std::string msg = std::string(what) + ": " + hcmx_gpu_last_error();
    if (status == HCMX_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    if (status == HCMX_CORRUPT_BUFFER) throw corrupt_buffer_error(msg);
    throw std::runtime_error(msg);
}

namespace codec {

enum class Scheme : std::uint8_t { afl = 0, aflp = 1, bfl = 2, dfl = 3 };  // codec.hpp:22

struct FormatDescriptor {  // codec.hpp:35-56
    Scheme scheme = Scheme::afl;
    std::uint8_t exp_bits = 2;
    std::uint8_t mant_bits = 2;
    double scale = 1.0;

    static unsigned alignment_unit(Scheme s) { return s == Scheme::afl ? 1u : s == Scheme::dfl ? 16u : 8u; }
    unsigned bit_width() const {
        const hcmx_descriptor d = raw();
        return hcmx_gpu_bit_width(&d);
    }
    hcmx_descriptor raw() const {
        hcmx_descriptor d{};
        d.scheme = static_cast<std::uint8_t>(scheme);
        d.exp_bits = exp_bits;
        d.mant_bits = mant_bits;
        d.bit_width = 0;
        d.scale = scale;
        d.bit_width = static_cast<std::uint8_t>(hcmx_gpu_bit_width(&d));
        return d;
    }
    static FormatDescriptor from(const hcmx_descriptor& d) {
        return {static_cast<Scheme>(d.scheme), d.exp_bits, d.mant_bits, d.scale};
    }
};

struct CompressedBuffer {  // codec.hpp:58-65
    FormatDescriptor descriptor;
    std::uint64_t count = 0;
    std::vector<std::uint8_t> payload;
    std::size_t byte_size() const { return 20 + payload.size(); }
};

struct BlockStats {  // codec.hpp:68-72
    double min_mag = 0.0;
    double max_mag = 0.0;
    bool all_zero = true;
};

inline constexpr std::size_t header_bytes = 20;

inline std::uint8_t mantissa_bits_for(double eps) {  // codec.cpp:62-67
    std::uint8_t m = 0;
    check(hcmx_gpu_mantissa_bits_for(eps, &m), "mantissa_bits_for");
    return m;
}

inline std::uint8_t exponent_bits_for(const BlockStats& s) {  // codec.cpp:69-79
    const hcmx_stats st{s.min_mag, s.max_mag, s.all_zero ? 1u : 0u, 0u};
    std::uint8_t e = 0;
    check(hcmx_gpu_exponent_bits_for(&st, &e), "exponent_bits_for");
    return e;
}

inline FormatDescriptor make_descriptor(Scheme scheme, double eps, const BlockStats& s) {  // codec.cpp:81-84
    const hcmx_stats st{s.min_mag, s.max_mag, s.all_zero ? 1u : 0u, 0u};
    hcmx_descriptor d{};
    check(hcmx_gpu_make_descriptor(static_cast<int>(scheme), eps, &st, &d), "make_descriptor");
    return FormatDescriptor::from(d);
}

inline FormatDescriptor make_descriptor(Scheme scheme, double eps, double scale,
                                        std::uint8_t exp_bits) {  // codec.cpp:86-101
    hcmx_descriptor d{};
    check(hcmx_gpu_make_descriptor_pinned(static_cast<int>(scheme), eps, scale, exp_bits, &d), "make_descriptor");
    return FormatDescriptor::from(d);
}

inline std::size_t compressed_size(std::uint64_t count, const FormatDescriptor& desc) {  // codec.cpp:179-181
    const hcmx_descriptor d = desc.raw();
    return static_cast<std::size_t>(hcmx_gpu_compressed_size(count, &d));
}

// codec.cpp:142-144 (analyze + layout + pack on the device)
inline CompressedBuffer compress(std::span<const double> values, double eps, Scheme scheme) {
    CompressedBuffer b;
    b.count = values.size();
    b.payload.resize(values.size() * 8 + 16);  // >= any layout's payload
    hcmx_descriptor d{};
    std::uint64_t len = 0;
    check(hcmx_gpu_compress(values.data(), values.size(), eps, static_cast<int>(scheme), &d, b.payload.data(),
                            b.payload.size(), &len),
          "compress");
    b.payload.resize(len);
    b.descriptor = FormatDescriptor::from(d);
    return b;
}

// codec.cpp:103-140
inline CompressedBuffer compress_block(std::span<const double> values, const FormatDescriptor& desc) {
    CompressedBuffer b;
    b.count = values.size();
    b.descriptor = desc;
    const hcmx_descriptor d = desc.raw();
    b.payload.resize(hcmx_gpu_payload_bytes(values.size(), &d) + 16);
    std::uint64_t len = 0;
    check(hcmx_gpu_compress_block(values.data(), values.size(), &d, b.payload.data(), b.payload.size(), &len),
          "compress_block");
    b.payload.resize(len);
    return b;
}

// codec.cpp:146-171
inline void decompress_into(const CompressedBuffer& buf, double* out) {
    const hcmx_descriptor d = buf.descriptor.raw();
    check(hcmx_gpu_decompress_into(&d, buf.count, buf.payload.data(), buf.payload.size(), out), "decompress_into");
}

inline std::vector<double> decompress(const CompressedBuffer& buf) {  // codec.cpp:173-177
    std::vector<double> out(buf.count);
    decompress_into(buf, out.data());
    return out;
}

// codec.cpp:187-225 wire format
inline void serialize(const CompressedBuffer& buf, std::vector<std::uint8_t>& out) {
    const hcmx_descriptor d = buf.descriptor.raw();
    const std::size_t at = out.size();
    out.resize(at + header_bytes + buf.payload.size());
    hcmx_gpu_serialize(&d, buf.count, buf.payload.data(), buf.payload.size(), out.data() + at);
}

inline CompressedBuffer deserialize(const std::uint8_t* data, std::size_t size, std::size_t& offset) {
    hcmx_descriptor d{};
    std::uint64_t off = offset, count = 0, at = 0, len = 0;
    check(hcmx_gpu_deserialize(data, size, &off, &d, &count, &at, &len), "deserialize");
    CompressedBuffer b;
    b.descriptor = FormatDescriptor::from(d);
    b.count = count;
    b.payload.assign(data + at, data + at + len);
    offset = static_cast<std::size_t>(off);
    return b;
}

}  // namespace codec

// Device-resident compressed H-matrix (hmatrix.hpp:51-78 flattened, see
// hcmx_hmat_desc) with the reference's matvec (hmatrix.hpp:126-128).
class DeviceHMatrix {
public:
    explicit DeviceHMatrix(const hcmx_hmat_desc& desc) : n_rows_(desc.n_rows), n_cols_(desc.n_cols) {
        check(hcmx_gpu_hmat_create(&desc, &h_), "hmat_create");
    }
    ~DeviceHMatrix() {
        if (h_) hcmx_gpu_hmat_destroy(h_);
    }
    DeviceHMatrix(const DeviceHMatrix&) = delete;
    DeviceHMatrix& operator=(const DeviceHMatrix&) = delete;

    // y := alpha * op(M) * x + beta * y (host vectors); transpose needs a matrix
    // created with desc.with_transpose = 1 (else std::invalid_argument)
    void matvec(double alpha, std::span<const double> x, double beta, std::span<double> y,
                bool transpose = false) const {
        if (x.size() != (transpose ? n_rows_ : n_cols_) || y.size() != (transpose ? n_cols_ : n_rows_))
            throw std::invalid_argument("matvec: dimension mismatch");
        check(hcmx_gpu_hmat_matvec(h_, alpha, x.data(), beta, y.data(), transpose ? 1 : 0), "matvec");
    }
    std::uint64_t rows() const { return n_rows_; }
    std::uint64_t cols() const { return n_cols_; }
    hcmx_memory_report memory() const {
        hcmx_memory_report r{};
        check(hcmx_gpu_hmat_memory(h_, &r), "memory");
        return r;
    }
    hcmx_hmat* handle() const { return h_; }

private:
    hcmx_hmat* h_ = nullptr;
    std::uint64_t n_rows_ = 0, n_cols_ = 0;
};

// hmatrix.hpp:126-128 as a free function (alpha == 0 leaves M untouched, a
// dimension mismatch throws std::invalid_argument)
inline void matvec(double alpha, const DeviceHMatrix& M, std::span<const double> x, double beta,
                   std::span<double> y, bool transpose = false) {
    M.matvec(alpha, x, beta, y, transpose);
}

#ifdef HCMX_GPU_HAVE_EIGEN
// the exact reference signature (hmatrix.hpp:127-128) where Eigen exists
inline void matvec(double alpha, const DeviceHMatrix& M, const Eigen::VectorXd& x, double beta,
                   Eigen::VectorXd& y, bool transpose = false) {
    M.matvec(alpha, std::span<const double>(x.data(), static_cast<std::size_t>(x.size())), beta,
             std::span<double>(y.data(), static_cast<std::size_t>(y.size())), transpose);
}
#endif

}  // namespace hcmx_gpu

#endif  // HCMX_GPU_HPP
