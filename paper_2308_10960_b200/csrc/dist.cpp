// dist.cpp -- block-row partitioning of a compressed H-matrix over the GPUs of
// one box behind the C-ABI: the partitioner, a partitioned handle
// that owns this rank's rows, and the exchange step of repeated products.
//
// The reference has no parallel code; its only hooks are the unused `threads`
// knobs (hmatrix.hpp:83,119) and SPEC's contract that disjoint leaf blocks may
// run concurrently with a deterministic merge.  Here every rank
// owns a contiguous row range: it builds only the leaves that write those rows
// (a lowrank leaf that crosses a cut is kept by both ranks, each doing the X^T x
// half for it), keeps x replicated and writes a disjoint slice of y -- nothing is
// reduced across ranks, so y is bit-identical to the single-GPU product.  The
// exchange that every rank needs before the next product is one NCCL group of
// in-place broadcasts (rank r sends rows [cut_r, cut_r+1)): an all-gather of
// unequal slices straight into a contiguous y, no padding, no staging copy.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2"), so the library has no
// link-time NCCL dependency and uses the NCCL the process already loaded
// (e.g. PyTorch's) when there is one.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <vector>

#include "internal.h"

namespace hcmx_gpu {
namespace {

// ---------------------------------------------------------------- NCCL ----
struct Nccl {
    void* so = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

struct nccl_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

const Nccl& nccl() {
    static std::once_flag once;
    static Nccl n;
    static std::string err;
    std::call_once(once, [] {
        n.so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!n.so) {
            err = std::string("NCCL not found: ") + dlerror();
            return;
        }
        auto sym = [&](const char* name) {
            void* p = dlsym(n.so, name);
            if (!p) err = std::string("NCCL symbol missing: ") + name;
            return p;
        };
        n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(sym("ncclGetUniqueId"));
        n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(sym("ncclCommInitRank"));
        n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
        n.CommCount = reinterpret_cast<decltype(n.CommCount)>(sym("ncclCommCount"));
        n.CommUserRank = reinterpret_cast<decltype(n.CommUserRank)>(sym("ncclCommUserRank"));
        n.Broadcast = reinterpret_cast<decltype(n.Broadcast)>(sym("ncclBroadcast"));
        n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(sym("ncclGroupStart"));
        n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(sym("ncclGroupEnd"));
        n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
    });
    if (!err.empty()) throw nccl_error(err);
    return n;
}

void check_nccl(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) {
        const Nccl& n = nccl();
        throw nccl_error(std::string(what) + ": " + (n.GetErrorString ? n.GetErrorString(r) : "NCCL error"));
    }
}

template <class F>
int guarded_nccl(F&& f) {
    try {
        f();
        return HCMX_OK;
    } catch (const nccl_error& e) {
        set_last_error(e.what());
        return HCMX_NCCL_ERROR;
    } catch (...) {
        return guarded([&] { throw; });
    }
}

// ----------------------------------------------------------- partitioner ----
// Contiguous row ranges, cut on multiples of 64 rows (leaf clusters of a
// power-of-two n), minimising the largest per-rank cost:
//   cost([a,b)) = sum over 64-row units of the phase-B bytes that land there
//                 (dense leaf and W-factor bytes, spread over each leaf's rows)
//               + the phase-A bytes (X factor + sigma) of EVERY lowrank leaf that
//                 overlaps [a,b) -- a leaf crossing a cut costs both ranks
// which is prefix(b) - prefix(a) + Xstart(b) - Xstart(a) + cross(a).  For a fixed
// start the cost grows with b, so the greedy sweep that extends each range as
// far as a bound B allows decides feasibility exactly; B is bisected.
std::vector<uint64_t> partition(const hcmx_hmat_desc& d, int world) {
    if (world < 1) throw invalid_argument("partition: world size must be >= 1");
    const uint64_t n = d.n_rows;
    constexpr uint64_t U = 64;
    const uint64_t nu = (n + U - 1) / U;
    auto plen = [&](int64_t b) { return static_cast<double>(d.plen[b]) + 20.0; };
    // per 64-row unit: phase-B bytes (spread over each leaf's rows); per lowrank
    // leaf: its phase-A bytes and the units it spans
    std::vector<double> ub(nu, 0.0);
    struct XLeaf {
        uint64_t first, last;
        double bytes;
    };
    std::vector<XLeaf> xleaves;
    for (uint64_t l = 0; l < d.nleaves; ++l) {
        const uint64_t r0 = static_cast<uint64_t>(d.row0[l]), r1 = static_cast<uint64_t>(d.row1[l]);
        double wbytes = 0.0, xbytes = 0.0;
        const int64_t k = d.rank[l];
        if (d.kind[l] == 0) {
            wbytes = plen(d.buf0[l]);
        } else if (d.kind[l] == 1) {
            for (int64_t i = 0; i < k; ++i) {
                wbytes += plen(d.buf0[l] + i);
                xbytes += plen(d.buf0[l] + k + i) + 8.0;
            }
        } else if (k > 0) {
            wbytes = plen(d.buf0[l]);
            xbytes = plen(d.buf0[l] + 1);
        }
        const double per_row = wbytes / static_cast<double>(r1 - r0);
        for (uint64_t u = r0 / U; u * U < r1; ++u) {
            const uint64_t a = std::max(r0, u * U), b = std::min(r1, (u + 1) * U);
            ub[u] += per_row * static_cast<double>(b - a);
        }
        if (xbytes > 0.0) xleaves.push_back({r0 / U, (r1 - 1) / U, xbytes});
    }
    // cb[u]: phase-B bytes of units [0, u); xs[u]: phase-A bytes of the leaves
    // starting before unit u; xcross[u]: those of the leaves spanning units u-1 and u
    std::vector<double> cb(nu + 1, 0.0), xs(nu + 1, 0.0), xcross(nu + 1, 0.0), xd(nu + 2, 0.0);
    for (uint64_t u = 0; u < nu; ++u) cb[u + 1] = cb[u] + ub[u];
    for (const XLeaf& x : xleaves) {
        xs[x.first + 1] += x.bytes;
        xd[x.first + 1] += x.bytes;
        xd[x.last + 1] -= x.bytes;
    }
    for (uint64_t u = 0; u < nu; ++u) xs[u + 1] += xs[u];
    double run = 0.0;
    for (uint64_t u = 0; u <= nu; ++u) {
        run += xd[u];
        xcross[u] = run;
    }
    auto cost = [&](uint64_t a, uint64_t b) { return cb[b] - cb[a] + xs[b] - xs[a] + xcross[a]; };
    // greedy sweep under bound B: number of ranges needed, and the cuts
    auto sweep = [&](double B, std::vector<uint64_t>* cuts) {
        uint64_t a = 0;
        int used = 0;
        if (cuts) cuts->assign(1, 0);
        while (a < nu) {
            // largest b > a with cost(a, b) <= B (at least one unit)
            uint64_t lo = a + 1, hi = nu;
            while (lo < hi) {
                const uint64_t mid = (lo + hi + 1) / 2;
                if (cost(a, mid) <= B) lo = mid;
                else hi = mid - 1;
            }
            a = lo;
            ++used;
            if (cuts) cuts->push_back(std::min<uint64_t>(a * U, n));
        }
        return used;
    };
    double lo = 0.0, hi = cost(0, nu);
    for (uint64_t u = 0; u < nu; ++u) lo = std::max(lo, cost(u, u + 1));
    for (int it = 0; it < 100 && hi - lo > 1e-9 * hi; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (sweep(mid, nullptr) <= world) hi = mid;
        else lo = mid;
    }
    std::vector<uint64_t> cuts;
    sweep(hi, &cuts);
    // fewer ranges than ranks (tiny matrices): split the largest ranges at unit
    // boundaries, else leave trailing ranks empty
    while (static_cast<int>(cuts.size()) - 1 < world) {
        size_t best = cuts.size();
        double bc = -1.0;
        for (size_t r = 0; r + 1 < cuts.size(); ++r) {
            const uint64_t a = cuts[r] / U, b = (cuts[r + 1] + U - 1) / U;
            if (b - a >= 2 && cost(a, b) > bc) {
                bc = cost(a, b);
                best = r;
            }
        }
        if (best == cuts.size()) {
            cuts.push_back(n);
            continue;
        }
        const uint64_t a = cuts[best] / U, b = (cuts[best + 1] + U - 1) / U;
        uint64_t m = a + 1;
        while (m + 1 < b && cost(a, m + 1) <= cost(m + 1, b)) ++m;
        cuts.insert(cuts.begin() + static_cast<long>(best) + 1, m * U);
    }
    cuts.back() = n;
    return cuts;
}

}  // namespace
}  // namespace hcmx_gpu

using namespace hcmx_gpu;

struct hcmx_hmat_dist {
    hcmx_hmat* local = nullptr;  // this rank's rows (nullptr: an empty range)
    ncclComm_t comm = nullptr;
    int world = 1, rank = 0;
    std::vector<uint64_t> cuts;
    uint64_t n_rows = 0, n_cols = 0;
    DevBuf xbuf, ybuf;
    cudaStream_t stream = nullptr;
};

namespace {

void exchange(hcmx_hmat_dist* h, double* d_y, cudaStream_t s) {
    if (h->world == 1) return;
    const Nccl& n = nccl();
    check_nccl(n.GroupStart(), "ncclGroupStart");
    for (int r = 0; r < h->world; ++r) {
        const uint64_t a = h->cuts[r], b = h->cuts[r + 1];
        if (b > a) check_nccl(n.Broadcast(d_y + a, d_y + a, b - a, ncclFloat64, r, h->comm, s), "ncclBroadcast");
    }
    check_nccl(n.GroupEnd(), "ncclGroupEnd");
}

void dist_matvec_device(hcmx_hmat_dist* h, double alpha, const double* d_x, double beta, double* d_y,
                        cudaStream_t s) {
    if (h->local) {
        const int st = hcmx_gpu_hmat_matvec_device(h->local, alpha, d_x, beta, d_y, s);
        if (st != HCMX_OK) throw cuda_error(std::string("partitioned matvec: ") + hcmx_gpu_last_error());
    }
    exchange(h, d_y, s);
}

}  // namespace

extern "C" {

int hcmx_gpu_partition_rows(const hcmx_hmat_desc* desc, int world, uint64_t* cuts) {
    return guarded([&] {
        if (!desc || !cuts) throw invalid_argument("partition: null argument");
        const std::vector<uint64_t> c = partition(*desc, world);
        std::copy(c.begin(), c.end(), cuts);
    });
}

int hcmx_gpu_nccl_unique_id(uint8_t* id128) {
    return guarded_nccl([&] {
        ncclUniqueId id;
        check_nccl(nccl().GetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(id128, id.internal, NCCL_UNIQUE_ID_BYTES);
    });
}

int hcmx_gpu_nccl_comm_init(int world, const uint8_t* id128, int rank, struct ncclComm** comm) {
    return guarded_nccl([&] {
        require_device();
        ncclUniqueId id;
        std::memcpy(id.internal, id128, NCCL_UNIQUE_ID_BYTES);
        check_nccl(nccl().CommInitRank(comm, world, id, rank), "ncclCommInitRank");
    });
}

int hcmx_gpu_nccl_comm_destroy(struct ncclComm* comm) {
    return guarded_nccl([&] {
        if (comm) check_nccl(nccl().CommDestroy(comm), "ncclCommDestroy");
    });
}

int hcmx_gpu_hmat_create_partitioned(const hcmx_hmat_desc* desc, struct ncclComm* comm, hcmx_hmat_dist** out) {
    return guarded_nccl([&] {
        require_device();
        auto* h = new hcmx_hmat_dist();
        try {
            h->comm = comm;
            if (comm) {
                check_nccl(nccl().CommCount(comm, &h->world), "ncclCommCount");
                check_nccl(nccl().CommUserRank(comm, &h->rank), "ncclCommUserRank");
            }
            h->n_rows = desc->n_rows;
            h->n_cols = desc->n_cols;
            h->cuts = partition(*desc, h->world);
            const uint64_t a = h->cuts[h->rank], b = h->cuts[h->rank + 1];
            if (b > a) {
                hcmx_hmat_desc d = *desc;
                d.row_begin = a;
                d.row_end = b;
                d.with_transpose = 0;
                const int st = hcmx_gpu_hmat_create(&d, &h->local);
                if (st != HCMX_OK) {
                    const std::string msg = hcmx_gpu_last_error();
                    if (st == HCMX_INVALID_ARGUMENT) throw invalid_argument(msg);
                    if (st == HCMX_CORRUPT_BUFFER) throw corrupt_buffer(msg);
                    if (st == HCMX_OUT_OF_MEMORY) throw oom_error(msg);
                    throw cuda_error(msg);
                }
            }
            check_cuda(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking), "cudaStreamCreate");
        } catch (...) {
            if (h->local) hcmx_gpu_hmat_destroy(h->local);
            if (h->stream) cudaStreamDestroy(h->stream);
            delete h;
            throw;
        }
        *out = h;
    });
}

int hcmx_gpu_hmat_dist_destroy(hcmx_hmat_dist* h) {
    return guarded([&] {
        if (!h) return;
        if (h->stream) cudaStreamSynchronize(h->stream);
        if (h->local) hcmx_gpu_hmat_destroy(h->local);
        if (h->stream) cudaStreamDestroy(h->stream);
        delete h;
    });
}

int hcmx_gpu_hmat_dist_rows(const hcmx_hmat_dist* h, uint64_t* row_begin, uint64_t* row_end, int* rank,
                            int* world) {
    return guarded([&] {
        if (row_begin) *row_begin = h->cuts[h->rank];
        if (row_end) *row_end = h->cuts[h->rank + 1];
        if (rank) *rank = h->rank;
        if (world) *world = h->world;
    });
}

int hcmx_gpu_hmat_dist_cuts(const hcmx_hmat_dist* h, uint64_t* cuts) {
    return guarded([&] { std::copy(h->cuts.begin(), h->cuts.end(), cuts); });
}

int hcmx_gpu_hmat_dist_local(hcmx_hmat_dist* h, hcmx_hmat** local) {
    return guarded([&] { *local = h->local; });
}

int hcmx_gpu_hmat_dist_matvec_device(hcmx_hmat_dist* h, double alpha, const double* d_x, double beta, double* d_y,
                                     void* stream) {
    return guarded_nccl([&] { dist_matvec_device(h, alpha, d_x, beta, d_y, static_cast<cudaStream_t>(stream)); });
}

int hcmx_gpu_hmat_dist_matvec(hcmx_hmat_dist* h, double alpha, const double* h_x, double beta, double* h_y) {
    return guarded_nccl([&] {
        cudaStream_t s = h->stream;
        if (!h->xbuf.p) h->xbuf.alloc(h->n_cols * 8);
        if (!h->ybuf.p) h->ybuf.alloc(h->n_rows * 8);
        h2d(h->xbuf.p, h_x, h->n_cols * 8, s);
        if (beta != 0.0) h2d(h->ybuf.p, h_y, h->n_rows * 8, s);
        dist_matvec_device(h, alpha, h->xbuf.as<double>(), beta, h->ybuf.as<double>(), s);
        d2h(h_y, h->ybuf.p, h->n_rows * 8, s);
        stream_sync(s);
    });
}

}  // extern "C"
