// kw_comm.cu — multi-GPU plumbing of the row-sharded DGEMM (one process per GPU).
//
// The reference is single-process and has no collective at all; the B200
// build adds exactly one: ncclBroadcast of DGEMM's B over NVLink 5 / NVSwitch.
// AXPY shards by index range and needs no communication.
//
// Row-sharded DGEMM: rank r owns row block r of A and C. B (k x n) lives on the root and is
// broadcast in column panels; panel j's broadcast (high-priority comm stream) overlaps the
// DGEMMs of earlier panels, which alternate between the queue's two compute streams so no panel
// ends in a partial wave. Each C element is reduced entirely on one rank by the single-GPU kernel in
// the same k order, so gathering the C row blocks reproduces the 1-GPU result bit for bit.
#include "kw_common.cuh"

#include <nccl.h>

#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <utility>
#include <vector>

namespace kw {
int dgemm_pick(size_t m, size_t n, size_t k);
size_t dgemm_krange_park_bytes(int cfg, size_t m, size_t n);
bool dgemm_krange_ok(size_t m, size_t n, size_t k, const double* A, size_t lda, const double* B, size_t ldb);
kw_status dgemm_device_krange(cudaStream_t s, int cfg, size_t m, size_t n, size_t k, double alpha, const double* A,
                              size_t lda, const double* B, size_t ldb, double beta, double* C, size_t ldc, int kt0,
                              int kt1, double* park);
kw_status dgemm_device_cfg(cudaStream_t s, int cfg, size_t m, size_t n, size_t k, double alpha, const double* A,
                           size_t lda, const double* B, size_t ldb, double beta, double* C, size_t ldc);
}

// NCCL is resolved at run time, never linked: a process that already loaded a libnccl.so.2
// (e.g. torch's bundled 2.28) keeps using that one (RTLD_NOLOAD), otherwise KW_NCCL_LIBRARY or
// the system libnccl.so.2 is opened. Linking it would pin the soname to whichever copy the
// loader finds first and break a later `import torch` that needs newer NCCL symbols.
namespace {
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    std::string error;
    bool ok = false;
};

NcclApi& nccl()
{
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        const char* env = std::getenv("KW_NCCL_LIBRARY");
        if (!h && env && *env)
            h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
        if (!h)
            h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            api.error = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
            return;
        }
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
        api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(dlsym(h, "ncclBroadcast"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
        api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Broadcast && api.GetErrorString;
        if (!api.ok)
            api.error = "libnccl.so.2 lacks a required symbol";
    });
    return api;
}

#define ncclGetUniqueId nccl().GetUniqueId
#define ncclCommInitRank nccl().CommInitRank
#define ncclCommDestroy nccl().CommDestroy
#define ncclBroadcast nccl().Broadcast
#define ncclGetErrorString nccl().GetErrorString

kw_status require_nccl()
{
    if (!nccl().ok)
        return kw::resource(nccl().error);
    return KW_OK;
}
} // namespace

struct kw_comm_s {
    ncclComm_t comm = nullptr;
    int device = 0, world = 1, rank = 0;
    cudaStream_t stream = nullptr; // broadcasts
    std::vector<cudaEvent_t> panel_ready;
    cudaEvent_t start = nullptr;
};

namespace {

kw_status nccl_fail(const char* what, ncclResult_t r)
{
    kw::set_error(std::string(what) + ": " + ncclGetErrorString(r));
    return KW_TASK;
}

// Column panels of B: [n0, n0 + w) pairs, equal widths of ceil(n / panels) rounded up to the
// 128-column tile. (A "head panel + one remainder" schedule measured slower on one GPU: the
// root's 2-D copy of the large remainder into the panel-major scratch was exposed —
// profiles/rowshard_rank_probe_r02.txt.) sharding.dgemm_panels mirrors this.
std::vector<std::pair<size_t, size_t>> panel_bounds(size_t n, int panels)
{
    const size_t tile = 128;
    const size_t w = kw::ceil_div(kw::ceil_div(n, static_cast<size_t>(panels)), tile) * tile;
    std::vector<std::pair<size_t, size_t>> out;
    for (size_t n0 = 0; n0 < n; n0 += w)
        out.emplace_back(n0, n - n0 < w ? n - n0 : w);
    return out;
}
size_t panel_ld(size_t wj) { return (wj + 7) & ~static_cast<size_t>(7); }

// Schedule of kw_dgemm_rowsharded (KW_ROWSHARD_SCHEDULE): "kslab" (default) broadcasts B in two
// row slabs — contiguous rows, so the root broadcasts straight from its own B (no packing copy
// when its pitch is the Buffer rule) — and runs the rank's product as two k-range launches (the
// first slab's k-tiles, accumulators parked; then the rest, reloaded): only the first slab's
// broadcast is exposed, the second overlaps the first pass, and each pass is one full
// data-parallel grid. "panels" = round 1's column panels with one launch per panel.
bool kslab_schedule()
{
    static const bool v = [] {
        const char* e = std::getenv("KW_ROWSHARD_SCHEDULE");
        return !(e && std::strcmp(e, "panels") == 0);
    }();
    return v;
}

// First slab of the k-slab schedule, in k-tiles of 16: 1/panels of the k-tiles (>= 1).
size_t first_slab_ktiles(size_t k, int panels)
{
    const size_t ktiles = kw::ceil_div(k, static_cast<size_t>(16));
    if (panels <= 1 || ktiles < 2)
        return ktiles;
    const size_t a = ktiles / static_cast<size_t>(panels);
    return a < 1 ? 1 : a;
}

kw_status ensure_events(kw_comm_s* c, int n)
{
    while (static_cast<int>(c->panel_ready.size()) < n) {
        cudaEvent_t e;
        cudaError_t err = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        if (err != cudaSuccess)
            return kw::cuda_fail("comm event", err);
        c->panel_ready.push_back(e);
    }
    return KW_OK;
}

} // namespace

namespace {
kw_status rowsharded_kslab(kw_comm_s* c, kw::Queue* q, size_t m_local, size_t n, size_t k, double alpha,
                           const double* A, size_t lda, const double* B, size_t ldb, double beta, double* C,
                           size_t ldc, double* scratch, int panels, int root)
{
    const size_t ldp = panel_ld(n);
    const size_t ktiles = kw::ceil_div(k, static_cast<size_t>(16));
    const bool is_root = c->rank == root;
    const bool direct = is_root && ldb == ldp; // the root broadcasts from (and computes on) B itself
    double* bmat = direct ? const_cast<double*>(B) : scratch;
    // Two passes need the TMA kernel (A with an even pitch, 16-byte aligned); otherwise one launch
    // after the whole broadcast (the library falls back to its cp.async kernel there).
    const size_t kt_a = kw::dgemm_krange_ok(m_local, n, k, A, lda, bmat, ldp) ? first_slab_ktiles(k, panels) : ktiles;
    const size_t rows_a = kt_a * 16 < k ? kt_a * 16 : k;
    const int cfg = kw::dgemm_pick(m_local, n, k);
    double* park = nullptr;
    if (kt_a < ktiles && m_local > 0) {
        kw_status st = kw::ensure_scratch(q, kw::dgemm_krange_park_bytes(cfg, m_local, n));
        if (st != KW_OK)
            return st;
        park = static_cast<double*>(q->scratch);
    }
    kw_status st = ensure_events(c, 2);
    if (st != KW_OK)
        return st;
    cudaError_t e = cudaEventRecord(c->start, q->stream); // B and C may come from earlier tasks
    if (e == cudaSuccess)
        e = cudaStreamWaitEvent(c->stream, c->start, 0);
    ncclResult_t r = ncclSuccess;
    if (k > 0 && e == cudaSuccess) {
        if (is_root && !direct)
            e = cudaMemcpy2DAsync(scratch, ldp * 8, B, ldb * 8, n * 8, k, cudaMemcpyDeviceToDevice, c->stream);
        // every rank, world 1 included, runs the broadcasts (in place at the root)
        if (e == cudaSuccess)
            r = ncclBroadcast(bmat, bmat, rows_a * ldp * sizeof(double), ncclChar, root, c->comm, c->stream);
        if (e == cudaSuccess && r == ncclSuccess)
            e = cudaEventRecord(c->panel_ready[0], c->stream);
        if (e == cudaSuccess && r == ncclSuccess && rows_a < k)
            r = ncclBroadcast(bmat + rows_a * ldp, bmat + rows_a * ldp, (k - rows_a) * ldp * sizeof(double), ncclChar,
                              root, c->comm, c->stream);
        if (e == cudaSuccess && r == ncclSuccess)
            e = cudaEventRecord(c->panel_ready[1], c->stream);
    }
    else if (e == cudaSuccess) {
        e = cudaEventRecord(c->panel_ready[0], c->stream);
        if (e == cudaSuccess)
            e = cudaEventRecord(c->panel_ready[1], c->stream);
    }
    if (r != ncclSuccess)
        return kw::task_fail(q, std::string("ncclBroadcast: ") + ncclGetErrorString(r));
    if (e == cudaSuccess)
        e = cudaStreamWaitEvent(q->stream, c->panel_ready[0], 0);
    if (e != cudaSuccess)
        return kw::task_fail(q, std::string("dgemm_rowsharded: ") + cudaGetErrorString(e));
    if (m_local > 0) {
        if (kt_a >= ktiles) {
            st = kw::dgemm_device_cfg(q->stream, cfg, m_local, n, k, alpha, A, lda, bmat, ldp, beta, C, ldc);
        }
        else {
            st = kw::dgemm_device_krange(q->stream, cfg, m_local, n, k, alpha, A, lda, bmat, ldp, beta, C, ldc, 0,
                                         static_cast<int>(kt_a), park);
            if (st == KW_OK) {
                e = cudaStreamWaitEvent(q->stream, c->panel_ready[1], 0);
                if (e != cudaSuccess)
                    return kw::task_fail(q, std::string("dgemm_rowsharded: ") + cudaGetErrorString(e));
                st = kw::dgemm_device_krange(q->stream, cfg, m_local, n, k, alpha, A, lda, bmat, ldp, beta, C, ldc,
                                             static_cast<int>(kt_a), static_cast<int>(ktiles), park);
            }
        }
        if (st != KW_OK)
            return kw::task_fail(q, kw::last_error());
    }
    // later tasks on the queue (and the next call's broadcasts into the scratch) follow both passes
    e = cudaStreamWaitEvent(q->stream, c->panel_ready[1], 0);
    if (e != cudaSuccess)
        return kw::task_fail(q, std::string("dgemm_rowsharded: ") + cudaGetErrorString(e));
    return kw::after_enqueue(q, "dgemm_rowsharded");
}
} // namespace

extern "C" {

kw_status kw_comm_unique_id(unsigned char id[128])
{
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    if (!id)
        return kw::usage("kw_comm_unique_id: null output");
    if (require_nccl() != KW_OK)
        return KW_RESOURCE;
    ncclUniqueId uid;
    ncclResult_t r = ncclGetUniqueId(&uid);
    if (r != ncclSuccess)
        return nccl_fail("ncclGetUniqueId", r);
    std::memcpy(id, &uid, sizeof(uid));
    return KW_OK;
}

kw_status kw_comm_init(kw_comm* out, int device, int world, int rank, const unsigned char id[128])
{
    if (!out || !id)
        return kw::usage("kw_comm_init: null argument");
    if (world < 1 || rank < 0 || rank >= world)
        return kw::usage("kw_comm_init: rank must lie in [0, world)");
    if (require_nccl() != KW_OK)
        return KW_RESOURCE;
    kw::DeviceGuard g(device);
    auto* c = new kw_comm_s;
    c->device = device;
    c->world = world;
    c->rank = rank;
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ncclResult_t r = ncclCommInitRank(&c->comm, world, uid, rank);
    if (r != ncclSuccess) {
        delete c;
        return nccl_fail("ncclCommInitRank", r);
    }
    // Highest priority: the broadcast kernels get SMs ahead of the queued GEMM CTAs, so panel
    // j+1 lands while panel j computes.
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaError_t e = cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, hi);
    if (e == cudaSuccess)
        e = cudaEventCreateWithFlags(&c->start, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        ncclCommDestroy(c->comm);
        delete c;
        return kw::cuda_fail("comm stream", e);
    }
    *out = c;
    return KW_OK;
}

kw_status kw_comm_destroy(kw_comm c)
{
    if (!c)
        return KW_OK;
    kw::DeviceGuard g(c->device);
    cudaStreamSynchronize(c->stream);
    for (cudaEvent_t e : c->panel_ready)
        cudaEventDestroy(e);
    cudaEventDestroy(c->start);
    cudaStreamDestroy(c->stream);
    ncclCommDestroy(c->comm);
    delete c;
    return KW_OK;
}

kw_status kw_comm_broadcast(kw_comm c, kw_queue qh, void* buf, size_t bytes, int root)
{
    KW_CHECK_QUEUE(qh);
    KW_ENQUEUE_LOCK(qh);
    if (!c)
        return kw::usage("kw_comm_broadcast: null communicator");
    if (root < 0 || root >= c->world)
        return kw::usage("kw_comm_broadcast: root out of range");
    auto* q = reinterpret_cast<kw::Queue*>(qh);
    kw::DeviceGuard g(q->device);
    ncclResult_t r = ncclBroadcast(buf, buf, bytes, ncclChar, root, c->comm, q->stream);
    if (r != ncclSuccess)
        return kw::task_fail(q, std::string("ncclBroadcast: ") + ncclGetErrorString(r));
    return kw::after_enqueue(q, "broadcast");
}

kw_status kw_dgemm_rowsharded_scratch(size_t n, size_t k, int panels, size_t* elems)
{
    if (!elems)
        return kw::usage("kw_dgemm_rowsharded_scratch: null output");
    if (panels < 1)
        return kw::usage("dgemm_rowsharded: panels must be >= 1");
    size_t total = 0;
    if (n > 0 && kslab_schedule())
        total = k * panel_ld(n); // B at the Buffer pitch rule
    else if (n > 0)
        for (const auto& b : panel_bounds(n, panels))
            total += k * panel_ld(b.second);
    *elems = total;
    return KW_OK;
}

kw_status kw_dgemm_rowsharded(kw_comm c, kw_queue qh, size_t m_local, size_t n, size_t k, double alpha,
                              const double* A, size_t lda, const double* B, size_t ldb, double beta, double* C,
                              size_t ldc, double* b_panels, int panels, int root)
{
    KW_CHECK_QUEUE(qh);
    KW_ENQUEUE_LOCK(qh);
    KW_NVTX("kw dgemm row-sharded");
    if (!c)
        return kw::usage("dgemm_rowsharded: null communicator");
    auto* q = reinterpret_cast<kw::Queue*>(qh);
    if (q->device != c->device)
        return kw::usage("dgemm_rowsharded: queue and communicator are on different devices");
    if (root < 0 || root >= c->world)
        return kw::usage("dgemm_rowsharded: root out of range");
    if (panels < 1)
        return kw::usage("dgemm_rowsharded: panels must be >= 1");
    if (n == 0)
        return KW_OK;
    if (!b_panels || (k > 0 && !A) || (m_local > 0 && !C))
        return kw::usage("dgemm_rowsharded: null buffer");
    if (c->rank == root && k > 0 && (!B || ldb < n))
        return kw::usage("dgemm_rowsharded: root needs B with ldb >= n");
    if (k > 0 && lda < k)
        return kw::usage("dgemm_rowsharded: lda smaller than k");
    if (m_local > 0 && ldc < n)
        return kw::usage("dgemm_rowsharded: ldc smaller than n");
    {
        // every operand (and the scratch) is device memory on the queue's device: a host or
        // foreign-device pointer would fault the context inside a copy or a kernel
        const void* ops[4] = {b_panels, k > 0 ? A : nullptr, m_local > 0 ? C : nullptr,
                              (c->rank == root && k > 0) ? B : nullptr};
        for (const void* ptr : ops) {
            int d = -1;
            if (ptr && (kw::pointer_kind(ptr, &d) != KW_MEM_DEVICE || d != q->device))
                return kw::usage("dgemm_rowsharded: operands and scratch must be device memory on the queue's device");
        }
    }
    if (kslab_schedule()) {
        kw::DeviceGuard g(q->device);
        return rowsharded_kslab(c, q, m_local, n, k, alpha, A, lda, B, ldb, beta, C, ldc, b_panels, panels, root);
    }
    // Panels start on 128-column tile boundaries (panel_bounds).
    const auto bounds = panel_bounds(n, panels);
    const int np = static_cast<int>(bounds.size());
    kw::DeviceGuard g(q->device);
    kw_status st = ensure_events(c, np);
    if (st != KW_OK)
        return st;
    cudaError_t e = cudaEventRecord(c->start, q->stream); // B and C may come from earlier tasks
    if (e == cudaSuccess)
        e = cudaStreamWaitEvent(c->stream, c->start, 0);
    // Panel launches alternate between the queue stream and its second compute stream: panel j+1's CTAs
    // fill the SMs while panel j's last wave drains (disjoint C columns, same per-element
    // arithmetic — bits unchanged). A panel launch ends in a partial wave otherwise: one rank's
    // 2048..8192-row block lost 2-13 % (tools/rowshard_rank_probe.py).
    if (e == cudaSuccess)
        e = cudaStreamWaitEvent(q->comp2, c->start, 0);
    ncclResult_t r = ncclSuccess;
    size_t off = 0;
    // One tile configuration for every panel launch of this rank — the one the whole m_local x n
    // product would get: panel grids that overlap on the two compute streams then co-reside
    // evenly (mixed 2- and 3-CTA/SM grids strand shared memory). Any paired configuration gives
    // the same bits.
    const int cfg = kw::dgemm_pick(m_local, n, k);
    for (int j = 0; j < np && e == cudaSuccess && r == ncclSuccess; ++j) {
        const size_t n0 = bounds[j].first, wj = bounds[j].second;
        // k x wj panel at the Buffer pitch rule (leading dimension a multiple of 8 doubles): an
        // odd-width last panel stays TMA-addressable, so it runs the same kernel (and k grouping)
        // as the resident 1-GPU launch — a dense odd pitch would drop to the cp.async kernel.
        const size_t ldp = panel_ld(wj);
        double* panel = b_panels + off;
        if (k > 0) {
            if (c->rank == root)
                e = cudaMemcpy2DAsync(panel, ldp * 8, B + n0, ldb * 8, wj * 8, k, cudaMemcpyDeviceToDevice, c->stream);
            // Every rank, world 1 included, runs the broadcast: a single-rank ncclBroadcast is legal
            // and keeps the one-GPU path the code path of the multi-GPU one.
            if (e == cudaSuccess)
                r = ncclBroadcast(panel, panel, k * ldp * sizeof(double), ncclChar, root, c->comm, c->stream);
        }
        if (e == cudaSuccess)
            e = cudaEventRecord(c->panel_ready[j], c->stream);
        cudaStream_t cs = (j & 1) ? q->comp2 : q->stream;
        if (e == cudaSuccess)
            e = cudaStreamWaitEvent(cs, c->panel_ready[j], 0);
        if (e == cudaSuccess && m_local > 0) {
            st = kw::dgemm_device_cfg(cs, cfg, m_local, wj, k, alpha, A, lda, panel, ldp, beta, C + n0, ldc);
            if (st != KW_OK)
                return kw::task_fail(q, kw::last_error());
        }
        off += k * ldp;
    }
    if (e == cudaSuccess)
        e = cudaEventRecord(q->ev_join2, q->comp2);
    if (e == cudaSuccess)
        e = cudaStreamWaitEvent(q->stream, q->ev_join2, 0);
    if (r != ncclSuccess)
        return kw::task_fail(q, std::string("ncclBroadcast: ") + ncclGetErrorString(r));
    if (e != cudaSuccess)
        return kw::task_fail(q, std::string("dgemm_rowsharded: ") + cudaGetErrorString(e));
    return kw::after_enqueue(q, "dgemm_rowsharded");
}

} // extern "C"
