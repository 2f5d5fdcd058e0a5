// compress.cu -- compress_in_place (hmatrix.hpp:115-119) behind
// the C-ABI: an assembled FP64 H-matrix in device memory (dense leaves, W, sigma,
// X of the lowrank leaves) -> the flattened compressed H-matrix (host tables +
// device blob) that hcmx_gpu_hmat_create takes, for every StorageMode kind
// (hmatrix.hpp:32-40):
//   aplr   dense -> codec::compress (iff dense_too, else FP64 words); lowrank ->
//          APLR, per-column precision from sigma (mixedprec.cpp:155-187)
//   codec  dense as above; lowrank U = W diag(sigma), V = X, one codec buffer
//          each (CodecLowrank, hmatrix.hpp:46-49)
//   mp     dense FP64 (MP never compresses dense); lowrank W Sigma X^H with its
//          columns in FP64 / FP32 / FP16 groups (mixedprec.cpp:66-120)
//   fp64   uncompressed: dense FP64, lowrank U, V in FP64 (LowrankBlock)
// The codec and APLR work runs on the device through the batched codec entry
// points; the host only lays out the tables.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "internal.h"

namespace hcmx_gpu {
namespace {

// U = W diag(sigma): column i (rows values) of every leaf scaled by sigma_i (one
// FP64 product per element, as U = W * sigma in the reference glue)
__global__ void k_scale_columns(const double* W, const uint64_t* off, const uint64_t* rows, const double* s,
                                uint64_t ncols, double* out) {
    for (uint64_t c = blockIdx.x; c < ncols; c += gridDim.x) {
        const uint64_t o = off[c], n = rows[c];
        const double v = s[c];
        for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) out[o + i] = __dmul_rn(W[o + i], v);
    }
}

// PackedSlice::pack (mixedprec.cpp:16-41): FP64 words as is, FP32 = (float)v,
// FP16 = float_to_half((float)v) (half.hpp: two round-to-nearest-even steps)
__global__ void k_pack_raw(const double* v, uint64_t n, int fmt, uint8_t* out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += gridDim.x * (uint64_t)blockDim.x) {
        if (fmt == HCMX_RAW_F64) {
            reinterpret_cast<double*>(out)[i] = v[i];
        } else if (fmt == HCMX_RAW_F32) {
            reinterpret_cast<float*>(out)[i] = __double2float_rn(v[i]);
        } else {
            reinterpret_cast<__half*>(out)[i] = __float2half_rn(__double2float_rn(v[i]));
        }
    }
}

constexpr double kMpRoundoff[3] = {1.1e-16, 6.0e-8, 4.9e-4};  // mixedprec.hpp:23 (MP-D-S-H)

inline uint64_t pad16(uint64_t x) { return (x + 15) & ~uint64_t(15); }

}  // namespace
}  // namespace hcmx_gpu

using namespace hcmx_gpu;

struct hcmx_flat {
    uint64_t n_rows = 0, n_cols = 0;
    std::vector<int64_t> row0, row1, col0, col1, kind, rank, buf0, sig0, count, poff, plen;
    std::vector<double> sigma;
    std::vector<hcmx_descriptor> desc;
    DevBuf blob;
    uint64_t blob_bytes = 0;
};

namespace {

hcmx_descriptor raw_desc(int fmt) {
    hcmx_descriptor d{};
    d.scheme = static_cast<uint8_t>(fmt);
    d.bit_width = static_cast<uint8_t>(fmt == HCMX_RAW_F64 ? 64 : fmt == HCMX_RAW_F32 ? 32 : 16);
    d.scale = 1.0;
    return d;
}

void check_status(int st) {
    if (st == HCMX_OK) return;
    const std::string m = hcmx_gpu_last_error();
    if (st == HCMX_INVALID_ARGUMENT) throw invalid_argument(m);
    if (st == HCMX_CORRUPT_BUFFER) throw corrupt_buffer(m);
    if (st == HCMX_OUT_OF_MEMORY) throw oom_error(m);
    throw cuda_error(m);
}

// codec::compress over buffers already laid end to end in device memory (the
// batched entry point); returns the payload arena and fills desc / poff
struct Compressed {
    DevBuf payload;
    std::vector<hcmx_descriptor> desc;
    std::vector<uint64_t> poff;
    uint64_t total = 0;
};

Compressed codec_batch(const double* d_values, const std::vector<uint64_t>& voff, const std::vector<uint64_t>& count,
                       double eps, int scheme, cudaStream_t s) {
    Compressed c;
    const uint64_t nb = count.size();
    c.desc.resize(nb);
    c.poff.resize(nb);
    uint64_t cap = 16;
    for (uint64_t b = 0; b < nb; ++b) cap += pad16(count[b] * 8);
    c.payload.alloc(cap);
    DevBuf dv(std::max<uint64_t>(16, nb * 8));
    h2d(dv.p, voff.data(), nb * 8, s);
    check_status(hcmx_gpu_codec_compress(d_values, dv.as<uint64_t>(), count.data(), nb, eps, scheme, c.payload.as<uint8_t>(),
                                         cap, c.desc.data(), c.poff.data(), &c.total, s));
    stream_sync(s);
    return c;
}

void compress_in_place(const hcmx_assembled& A, double eps, int storage, int scheme, int dense_too, hcmx_flat* f,
                       cudaStream_t s) {
    if (storage < HCMX_STORE_APLR || storage > HCMX_STORE_FP64) throw invalid_argument("compress_in_place: storage mode");
    if (storage != HCMX_STORE_FP64) alignment_unit(scheme);  // scheme validation
    const uint64_t L = A.nleaves;
    f->n_rows = A.n_rows;
    f->n_cols = A.n_cols;
    f->row0.assign(A.row0, A.row0 + L);
    f->row1.assign(A.row1, A.row1 + L);
    f->col0.assign(A.col0, A.col0 + L);
    f->col1.assign(A.col1, A.col1 + L);
    f->kind.assign(L, 0);
    f->rank.assign(L, 0);
    f->buf0.assign(L, 0);
    f->sig0.assign(L, 0);
    const bool uniform = storage == HCMX_STORE_CODEC || storage == HCMX_STORE_FP64;  // lowrank as U, V (kind 2)
    std::vector<uint64_t> nbuf(L);
    uint64_t nb = 0;
    for (uint64_t l = 0; l < L; ++l) {
        const int64_t k = A.rank[l];
        if (A.kind[l] != 0 && A.kind[l] != 1) throw invalid_argument("compress_in_place: leaf kind must be 0 (dense) or 1 (lowrank)");
        if (k < 0) throw invalid_argument("compress_in_place: negative rank");
        f->kind[l] = A.kind[l] == 0 ? 0 : (uniform ? 2 : 1);
        f->rank[l] = A.kind[l] == 0 ? 0 : k;
        nbuf[l] = A.kind[l] == 0 ? 1 : (uniform ? (k > 0 ? 2 : 0) : 2 * static_cast<uint64_t>(k));
        f->buf0[l] = static_cast<int64_t>(nb);
        nb += nbuf[l];
    }
    f->desc.assign(nb, hcmx_descriptor{});
    f->count.assign(nb, 0);
    f->poff.assign(nb, 0);
    f->plen.assign(nb, 0);
    std::vector<uint64_t> at(nb, 0);       // byte offset of each buffer's payload inside its part
    std::vector<int> part_of(nb, -1);
    std::vector<DevBuf> parts;
    std::vector<uint64_t> part_bytes;
    auto rows = [&](uint64_t l) { return static_cast<uint64_t>(A.row1[l] - A.row0[l]); };
    auto cols = [&](uint64_t l) { return static_cast<uint64_t>(A.col1[l] - A.col0[l]); };

    // ---- dense leaves
    std::vector<uint64_t> didx;
    for (uint64_t l = 0; l < L; ++l)
        if (A.kind[l] == 0) didx.push_back(l);
    if (!didx.empty()) {
        std::vector<uint64_t> voff, cnt;
        for (uint64_t l : didx) {
            voff.push_back(static_cast<uint64_t>(A.dense_off[l]));
            cnt.push_back(rows(l) * cols(l));
        }
        const bool codec = (storage == HCMX_STORE_APLR || storage == HCMX_STORE_CODEC) && dense_too;
        if (codec) {
            Compressed c = codec_batch(A.d_dense, voff, cnt, eps, scheme, s);
            for (size_t i = 0; i < didx.size(); ++i) {
                const uint64_t b = f->buf0[didx[i]];
                f->desc[b] = c.desc[i];
                f->count[b] = static_cast<int64_t>(cnt[i]);
                at[b] = c.poff[i];
                part_of[b] = static_cast<int>(parts.size());
            }
            part_bytes.push_back(c.total);
            parts.push_back(std::move(c.payload));
        } else {  // FP64 words (StorageMode fp64 / mp, or dense_too = false)
            uint64_t tot = 0;
            for (size_t i = 0; i < didx.size(); ++i) tot += cnt[i] * 8;
            DevBuf raw(std::max<uint64_t>(16, tot));
            uint64_t o = 0;
            for (size_t i = 0; i < didx.size(); ++i) {
                check_cuda(cudaMemcpyAsync(raw.as<uint8_t>() + o, A.d_dense + voff[i], cnt[i] * 8, cudaMemcpyDeviceToDevice, s),
                           "dense copy");
                const uint64_t b = f->buf0[didx[i]];
                f->desc[b] = raw_desc(HCMX_RAW_F64);
                f->count[b] = static_cast<int64_t>(cnt[i]);
                at[b] = o;
                part_of[b] = static_cast<int>(parts.size());
                o += cnt[i] * 8;
            }
            part_bytes.push_back(tot);
            parts.push_back(std::move(raw));
        }
    }

    // ---- lowrank leaves
    std::vector<uint64_t> lidx;
    for (uint64_t l = 0; l < L; ++l)
        if (A.kind[l] == 1 && A.rank[l] > 0) lidx.push_back(l);
    if (storage == HCMX_STORE_APLR && !lidx.empty()) {
        std::vector<uint64_t> r, c, k, wo, xo, so, bo;
        uint64_t nlb = 0, cap = 16;
        for (uint64_t l : lidx) {
            r.push_back(rows(l));
            c.push_back(cols(l));
            k.push_back(static_cast<uint64_t>(A.rank[l]));
            wo.push_back(static_cast<uint64_t>(A.w_off[l]));
            xo.push_back(static_cast<uint64_t>(A.x_off[l]));
            so.push_back(static_cast<uint64_t>(A.sig_off[l]));
            bo.push_back(nlb);
            nlb += 2 * k.back();
            cap += (r.back() + c.back()) * k.back() * 8 + 2 * k.back() * 16;
        }
        DevBuf pay(cap);
        std::vector<hcmx_descriptor> d(nlb);
        std::vector<uint64_t> po(nlb);
        uint64_t tot = 0;
        check_status(hcmx_gpu_aplr_compress(lidx.size(), r.data(), c.data(), k.data(), A.d_W, wo.data(), A.d_X, xo.data(),
                                            A.sigma, so.data(), bo.data(), eps, scheme, pay.as<uint8_t>(), cap, d.data(),
                                            po.data(), &tot, s));
        for (size_t i = 0; i < lidx.size(); ++i) {
            const uint64_t l = lidx[i], kk = k[i];
            for (uint64_t j = 0; j < 2 * kk; ++j) {
                const uint64_t b = f->buf0[l] + j;
                f->desc[b] = d[bo[i] + j];
                f->count[b] = static_cast<int64_t>(j < kk ? r[i] : c[i]);
                at[b] = po[bo[i] + j];
                part_of[b] = static_cast<int>(parts.size());
            }
        }
        part_bytes.push_back(tot);
        parts.push_back(std::move(pay));
    } else if (uniform && !lidx.empty()) {
        // U = W diag(sigma) (device), V = X: values end to end, then one codec
        // buffer (or FP64 words) each
        uint64_t tot = 0;
        std::vector<uint64_t> voff, cnt, colo, colr;
        std::vector<double> colsig;
        for (uint64_t l : lidx) {
            const uint64_t kk = static_cast<uint64_t>(A.rank[l]);
            voff.push_back(tot);
            cnt.push_back(rows(l) * kk);
            for (uint64_t i = 0; i < kk; ++i) {
                colo.push_back(tot + i * rows(l));
                colr.push_back(rows(l));
                colsig.push_back(A.sigma[A.sig_off[l] + i]);
            }
            tot += rows(l) * kk;
            voff.push_back(tot);
            cnt.push_back(cols(l) * kk);
            tot += cols(l) * kk;
        }
        DevBuf vals(std::max<uint64_t>(16, tot * 8));
        std::vector<uint64_t> srco;  // W column offsets in the assembled arrays
        for (uint64_t l : lidx)
            for (int64_t i = 0; i < A.rank[l]; ++i) srco.push_back(static_cast<uint64_t>(A.w_off[l]) + i * rows(l));
        // copy W (then scale in place) and X into the value array
        for (size_t i = 0; i < lidx.size(); ++i) {
            const uint64_t l = lidx[i], kk = static_cast<uint64_t>(A.rank[l]);
            check_cuda(cudaMemcpyAsync(vals.as<double>() + voff[2 * i], A.d_W + A.w_off[l], rows(l) * kk * 8,
                                       cudaMemcpyDeviceToDevice, s), "W copy");
            check_cuda(cudaMemcpyAsync(vals.as<double>() + voff[2 * i + 1], A.d_X + A.x_off[l], cols(l) * kk * 8,
                                       cudaMemcpyDeviceToDevice, s), "X copy");
        }
        {
            const uint64_t nc = colo.size();
            DevBuf dco(nc * 8), dcr(nc * 8), dcs(nc * 8);
            h2d(dco.p, colo.data(), nc * 8, s);
            h2d(dcr.p, colr.data(), nc * 8, s);
            h2d(dcs.p, colsig.data(), nc * 8, s);
            k_scale_columns<<<(int)std::min<uint64_t>(nc, 65535), 128, 0, s>>>(vals.as<double>(), dco.as<uint64_t>(),
                                                                              dcr.as<uint64_t>(), dcs.as<double>(), nc,
                                                                              vals.as<double>());
            check_cuda(cudaGetLastError(), "scale launch");
            stream_sync(s);
        }
        if (storage == HCMX_STORE_CODEC) {
            Compressed c = codec_batch(vals.as<double>(), voff, cnt, eps, scheme, s);
            for (size_t i = 0; i < lidx.size(); ++i)
                for (int j = 0; j < 2; ++j) {
                    const uint64_t b = f->buf0[lidx[i]] + j;
                    f->desc[b] = c.desc[2 * i + j];
                    f->count[b] = static_cast<int64_t>(cnt[2 * i + j]);
                    at[b] = c.poff[2 * i + j];
                    part_of[b] = static_cast<int>(parts.size());
                }
            part_bytes.push_back(c.total);
            parts.push_back(std::move(c.payload));
        } else {
            for (size_t i = 0; i < lidx.size(); ++i)
                for (int j = 0; j < 2; ++j) {
                    const uint64_t b = f->buf0[lidx[i]] + j;
                    f->desc[b] = raw_desc(HCMX_RAW_F64);
                    f->count[b] = static_cast<int64_t>(cnt[2 * i + j]);
                    at[b] = voff[2 * i + j] * 8;
                    part_of[b] = static_cast<int>(parts.size());
                }
            part_bytes.push_back(tot * 8);
            parts.push_back(std::move(vals));
        }
    } else if (storage == HCMX_STORE_MP && !lidx.empty()) {
        // mp_partition (mixedprec.cpp:66-82): per column the cheapest of FP64 /
        // FP32 / FP16 whose unit roundoff keeps sigma_j * rho <= delta = eps sigma_0
        uint64_t tot = 0;
        struct Job {
            const double* src;
            uint64_t n, dst;
            int fmt;
        };
        std::vector<Job> jobs;
        for (uint64_t l : lidx) {
            const int64_t kk = A.rank[l];
            const double* sg = A.sigma + A.sig_off[l];
            const double delta = eps * sg[0];
            int prev = 0;
            for (int64_t i = 0; i < kk; ++i) {
                int g = 0;
                if (sg[i] * kMpRoundoff[1] <= delta) g = 1;
                if (sg[i] * kMpRoundoff[2] <= delta) g = 2;
                if (sg[i] <= delta) throw invalid_argument("compress_in_place: mp needs sigma above eps * sigma_0");
                if (g < prev) throw invalid_argument("compress_in_place: mp needs decreasing sigma");
                prev = g;
                const int fmt = HCMX_RAW_F64 + g;
                const uint64_t wb = f->buf0[l] + i, xb = f->buf0[l] + kk + i;
                const unsigned bytes = fmt == HCMX_RAW_F64 ? 8 : fmt == HCMX_RAW_F32 ? 4 : 2;
                for (int side = 0; side < 2; ++side) {
                    const uint64_t b = side ? xb : wb, n = side ? cols(l) : rows(l);
                    const double* src = side ? A.d_X + A.x_off[l] + i * cols(l) : A.d_W + A.w_off[l] + i * rows(l);
                    f->desc[b] = raw_desc(fmt);
                    f->count[b] = static_cast<int64_t>(n);
                    at[b] = tot;
                    part_of[b] = static_cast<int>(parts.size());
                    jobs.push_back({src, n, tot, fmt});
                    tot += pad16(n * bytes);
                }
            }
        }
        DevBuf raw(std::max<uint64_t>(16, tot));
        for (const Job& j : jobs)
            k_pack_raw<<<(int)std::min<uint64_t>((j.n + 255) / 256, 1024), 256, 0, s>>>(j.src, j.n, j.fmt,
                                                                                        raw.as<uint8_t>() + j.dst);
        check_cuda(cudaGetLastError(), "pack launch");
        part_bytes.push_back(tot);
        parts.push_back(std::move(raw));
    }

    // ---- one blob: the parts back to back, 16-byte aligned
    std::vector<uint64_t> base(parts.size(), 0);
    uint64_t total = 0;
    for (size_t q = 0; q < parts.size(); ++q) {
        base[q] = total;
        total += pad16(part_bytes[q]);
    }
    // the parts were sized for the worst case (FP64 words): keep only their used
    // bytes before the blob is allocated, so the peak stays near the compressed size
    for (size_t q = 0; q < parts.size(); ++q) {
        if (parts[q].bytes > pad16(part_bytes[q]) + (64u << 20)) {
            DevBuf tight(std::max<uint64_t>(16, part_bytes[q]));
            if (part_bytes[q])
                check_cuda(cudaMemcpyAsync(tight.p, parts[q].p, part_bytes[q], cudaMemcpyDeviceToDevice, s), "part copy");
            stream_sync(s);
            parts[q] = std::move(tight);
        }
    }
    f->blob.alloc(std::max<uint64_t>(16, total));
    for (size_t q = 0; q < parts.size(); ++q) {
        if (part_bytes[q])
            check_cuda(cudaMemcpyAsync(f->blob.as<uint8_t>() + base[q], parts[q].p, part_bytes[q], cudaMemcpyDeviceToDevice, s),
                       "blob copy");
        stream_sync(s);
        parts[q].release();
    }
    f->blob_bytes = total;
    for (uint64_t b = 0; b < nb; ++b) {
        if (part_of[b] < 0) throw std::logic_error("compress_in_place: buffer without payload");
        f->poff[b] = static_cast<int64_t>(base[part_of[b]] + at[b]);
        f->plen[b] = static_cast<int64_t>(payload_bytes(f->count[b], f->desc[b].bit_width));
    }
    // sigma: APLR / MP leaves keep theirs (sig0 into the caller's array); U V^T leaves need none
    uint64_t nsig = 0;
    for (uint64_t l = 0; l < L; ++l)
        if (f->kind[l] == 1) nsig = std::max<uint64_t>(nsig, static_cast<uint64_t>(A.sig_off[l] + A.rank[l]));
    f->sigma.assign(A.sigma, A.sigma + nsig);
    if (f->sigma.empty()) f->sigma.push_back(0.0);
    for (uint64_t l = 0; l < L; ++l) f->sig0[l] = f->kind[l] == 1 ? A.sig_off[l] : 0;
}

void report_of(const hcmx_flat& f, hcmx_memory_report* r) {
    *r = hcmx_memory_report{};
    for (size_t l = 0; l < f.row0.size(); ++l) {
        const uint64_t rows = f.row1[l] - f.row0[l], cols = f.col1[l] - f.col0[l];
        const int64_t b0 = f.buf0[l], k = f.rank[l];
        auto bytes = [&](int64_t b) {
            const bool raw = f.desc[b].scheme >= HCMX_RAW_F64;
            return static_cast<uint64_t>(f.plen[b]) + (raw ? 0 : 20);
        };
        if (f.kind[l] == 0) {
            r->dense_leaves++;
            r->uncompressed_equivalent += 8 * rows * cols;
            if (f.desc[b0].scheme >= HCMX_RAW_F64) r->dense_raw += f.plen[b0];
            else r->dense_compressed += bytes(b0);
        } else {
            r->lowrank_leaves++;
            r->uncompressed_equivalent += 8 * (rows + cols) * k;
            uint64_t t = f.kind[l] == 1 ? 8 + 8 * k : 4;
            const int64_t nbuf = f.kind[l] == 1 ? 2 * k : (k > 0 ? 2 : 0);
            for (int64_t j = 0; j < nbuf; ++j) t += bytes(b0 + j);
            r->lowrank_compressed += t;
        }
    }
    r->overhead = 16 * f.row0.size();
}

}  // namespace

extern "C" {

int hcmx_gpu_compress_in_place(const hcmx_assembled* A, double eps, int storage, int scheme, int dense_too,
                               hcmx_flat** out, hcmx_memory_report* report, void* stream) {
    return guarded([&] {
        require_device();
        auto* f = new hcmx_flat();
        try {
            compress_in_place(*A, eps, storage, scheme, dense_too, f, static_cast<cudaStream_t>(stream));
        } catch (...) {
            delete f;
            throw;
        }
        if (report) report_of(*f, report);
        *out = f;
    });
}

int hcmx_gpu_flat_desc(const hcmx_flat* f, hcmx_hmat_desc* d) {
    return guarded([&] {
        *d = hcmx_hmat_desc{};
        d->n_rows = f->n_rows;
        d->n_cols = f->n_cols;
        d->nleaves = f->row0.size();
        d->nbuffers = f->desc.size();
        d->nsigma = f->sigma.size();
        d->blob_bytes = f->blob_bytes;
        d->row0 = f->row0.data();
        d->row1 = f->row1.data();
        d->col0 = f->col0.data();
        d->col1 = f->col1.data();
        d->kind = f->kind.data();
        d->rank = f->rank.data();
        d->buf0 = f->buf0.data();
        d->sig0 = f->sig0.data();
        d->sigma = f->sigma.data();
        d->desc = f->desc.data();
        d->count = f->count.data();
        d->poff = f->poff.data();
        d->plen = f->plen.data();
        d->blob = f->blob.as<uint8_t>();
        d->blob_on_device = 1;
    });
}

int hcmx_gpu_flat_copy_blob(const hcmx_flat* f, uint8_t* d_dst, void* stream) {
    return guarded([&] {
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        if (f->blob_bytes)
            check_cuda(cudaMemcpyAsync(d_dst, f->blob.p, f->blob_bytes, cudaMemcpyDeviceToDevice, s), "blob copy");
        stream_sync(s);
    });
}

int hcmx_gpu_flat_destroy(hcmx_flat* f) {
    return guarded([&] { delete f; });
}

}  // extern "C"
