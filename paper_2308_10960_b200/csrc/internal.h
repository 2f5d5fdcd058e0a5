// internal.h -- shared declarations of libhcmx_gpu (not part of the C-ABI).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "hcmx_gpu.h"

namespace hcmx_gpu {

// error plumbing: C++ exceptions inside the library, statuses at the C-ABI
struct invalid_argument : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct corrupt_buffer : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct cuda_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct oom_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void set_last_error(const std::string& s);

template <class F>
int guarded(F&& f) {
    try {
        f();
        return HCMX_OK;
    } catch (const invalid_argument& e) {
        set_last_error(e.what());
        return HCMX_INVALID_ARGUMENT;
    } catch (const corrupt_buffer& e) {
        set_last_error(e.what());
        return HCMX_CORRUPT_BUFFER;
    } catch (const oom_error& e) {
        set_last_error(e.what());
        return HCMX_OUT_OF_MEMORY;
    } catch (const cuda_error& e) {
        set_last_error(e.what());
        return HCMX_CUDA_ERROR;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return HCMX_CUDA_ERROR;
    }
}

// ---- scalar layout rules (codec_host.cpp; reference codec.cpp:25-101) ----
unsigned alignment_unit(int scheme);
unsigned bit_width(int scheme, unsigned e, unsigned m);
uint8_t mantissa_bits_for(double eps);
uint8_t exponent_bits_for(const hcmx_stats& st);
hcmx_descriptor make_descriptor(int scheme, double eps, double scale, uint8_t exp_bits);
hcmx_descriptor make_descriptor(int scheme, double eps, const hcmx_stats& st);
inline uint64_t payload_bytes(uint64_t count, unsigned w) { return (count * w + 7) / 8; }
inline uint64_t round16(uint64_t x) { return (x + 15) & ~uint64_t(15); }

// ---- device codec launchers (codec_kernels.cu); d_count is the device copy of h_count ----
void launch_analyze_jobs(const double* values, const uint64_t* voff, const uint64_t* d_count,
                         const uint64_t* h_count, uint64_t nbuf, hcmx_stats* stats, void* stream);
int launch_pack_jobs(const double* values, const uint64_t* voff, const uint64_t* d_count,
                     const uint64_t* h_count, const hcmx_descriptor* desc, const uint64_t* poff,
                     uint64_t nbuf, uint8_t* payload, void* stream);
void launch_unpack_jobs(const uint8_t* payload, const uint64_t* poff, const uint64_t* d_count,
                        const uint64_t* h_count, const hcmx_descriptor* desc, const uint64_t* voff,
                        uint64_t nbuf, double* out, void* stream);

void check_cuda(int err, const char* what);  // err is a cudaError_t
void require_device();

// RAII device buffer
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    explicit DevBuf(size_t n) { alloc(n); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) { release(); p = o.p; bytes = o.bytes; o.p = nullptr; o.bytes = 0; }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t n);
    void release();
    template <class T> T* as() const { return static_cast<T*>(p); }
};

void h2d(void* dst, const void* src, size_t bytes, void* stream);
void d2h(void* dst, const void* src, size_t bytes, void* stream);
void stream_sync(void* stream);

}  // namespace hcmx_gpu
