// kw_dgemm_e2e.cu — DGEMM on host-resident operands (the e2e path of kw_dgemm / GemmTiledKernel
// on Device::host() buffers): the row-panel ring schedule and the streamed square-growth
// schedule feeding one persistent launch (DESIGN.md §4 "e2e DGEMM"). Both run the same kernels
// as the resident launch, so the results are bitwise those of the resident launch.
#include "kw_dgemm_internal.cuh"

#include <cuda.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

namespace kw::gemm {

// Host-resident operands (e2e path): B is staged once, then row panels of A and C stream
// through a three-slot ring on three streams — H2D(A_p, C_p) on the copy stream, DGEMM on the
// queue stream, D2H(C_p) on the aux stream — so panel p+1's upload, panel p's compute and
// panel p-1's download overlap (PCIe is full duplex). Each C element is produced by the same
// kernel in the same k order, so panelling changes no bit.
kw_status dgemm_staged(kw::Queue* q, int tile, size_t m, size_t n, size_t k, double alpha, const double* A,
                       size_t lda, const double* B, size_t ldb, double beta, double* C, size_t ldc, bool a_dev,
                       bool b_dev, bool c_dev)
{
    KW_NVTX("kw dgemm e2e: row panels");
    const size_t ldbs = round2(n), ldas = round2(k == 0 ? 1 : k), ldcs = round2(n);
    const size_t row_bytes = (ldas + ldcs) * sizeof(double);
    // Panel height: about m/16 in whole 64-row tiles (the launcher sizes its CTA tile to the
    // panel, so small panels still fill the GPU), capped at 1 GiB per slot. Sixteen panels keep
    // the pipeline fill (first upload) and drain (last compute + download) short; measured best
    // or tied at 4096 and 8192 among 256..4096-row panels (profiles/e2e_dgemm_panel_sweep_r01.txt).
    size_t R = kw::ceil_div(kw::ceil_div(m, static_cast<size_t>(16)), 64) * 64;
    const size_t cap = std::max<size_t>(64, ((1ull << 30) / row_bytes) / 64 * 64);
    R = std::min(std::max<size_t>(R, 64), cap);
    if (R > m)
        R = m;
    const int ring = 3;
    const size_t b_bytes = b_dev ? 0 : k * ldbs * sizeof(double);
    const size_t slot_bytes = R * row_bytes;
    kw_status st = kw::ensure_scratch(q, b_bytes + ring * slot_bytes + 256);
    if (st != KW_OK)
        return st;
    char* base = static_cast<char*>(q->scratch);
    const double* Bd = B;
    size_t ldbd = ldb;
    // Earlier work on the queue (which may produce A/B/C) precedes the uploads.
    cudaError_t e = cudaEventRecord(q->ev_start, q->stream);
    if (e == cudaSuccess)
        e = cudaStreamWaitEvent(q->h2d, q->ev_start, 0);
    if (e == cudaSuccess)
        e = cudaStreamWaitEvent(q->comp2, q->ev_start, 0);
    // B streaming: B is uploaded in column panels into its dense device copy; the first row
    // panel is computed block by block as the B panels land, the remaining row panels (full
    // width) after the last one. Start latency = A_0 + C_0 + one B panel instead of all of B.
    const bool stream_b = !b_dev && k > 0;
    int nbp = 0;
    size_t bw = n;
    if (stream_b) {
        bw = kw::ceil_div(kw::ceil_div(n, static_cast<size_t>(4)), 128) * 128;
        nbp = static_cast<int>(kw::ceil_div(n, bw));
        if (nbp > kw::Queue::kBPanels) {
            bw = kw::ceil_div(n, static_cast<size_t>(kw::Queue::kBPanels));
            bw = kw::ceil_div(bw, 128) * 128;
            nbp = static_cast<int>(kw::ceil_div(n, bw));
        }
        Bd = reinterpret_cast<double*>(base);
        ldbd = ldbs;
    }
    char* slots = base + ((b_bytes + 255) / 256) * 256;
    const size_t npanels = kw::ceil_div(m, R);
    // KW_E2E_TRACE: CUDA-event timeline (start, B resident, last upload, last compute, last download)
    const bool trace = std::getenv("KW_E2E_TRACE") != nullptr;
    cudaEvent_t tev[5] = {};
    if (trace) {
        for (auto& ev : tev)
            cudaEventCreate(&ev);
        cudaEventRecord(tev[0], q->stream);
    }
    for (size_t pi = 0; pi < npanels && e == cudaSuccess; ++pi) {
        const int s = static_cast<int>(pi % ring);
        const size_t r0 = pi * R, rows = m - r0 < R ? m - r0 : R;
        // Odd panels compute on the second stream: a panel launch is a fraction of a wave at
        // these heights, so consecutive panels overlap instead of each ending in a tail.
        cudaStream_t comp = (pi & 1) ? q->comp2 : q->stream;
        double* as = reinterpret_cast<double*>(slots + s * slot_bytes);
        double* cs = as + R * ldas;
        if (pi >= static_cast<size_t>(ring))
            e = cudaStreamWaitEvent(q->h2d, q->ev_free[s], 0);
        const double* Ad = A + r0 * lda;
        size_t ldad = lda;
        double* Cd = C + r0 * ldc;
        size_t ldcd = ldc;
        bool uploaded = false;
        if (e == cudaSuccess && !a_dev && k > 0) {
            e = cudaMemcpy2DAsync(as, ldas * 8, A + r0 * lda, lda * 8, k * 8, rows, cudaMemcpyHostToDevice, q->h2d);
            Ad = as;
            ldad = ldas;
            uploaded = true;
        }
        if (e == cudaSuccess && !c_dev) {
            e = cudaMemcpy2DAsync(cs, ldcs * 8, C + r0 * ldc, ldc * 8, n * 8, rows, cudaMemcpyHostToDevice, q->h2d);
            Cd = cs;
            ldcd = ldcs;
            uploaded = true;
        }
        if (e == cudaSuccess && uploaded) {
            e = cudaEventRecord(q->ev_h2d[s], q->h2d);
            if (e == cudaSuccess)
                e = cudaStreamWaitEvent(comp, q->ev_h2d[s], 0);
        }
        if (e != cudaSuccess)
            break;
        if (pi == 0 && stream_b) {
            // B column panels behind the first A/C panel on the copy stream; compute block (0, j)
            // as soon as panel j is resident.
            for (int j = 0; j < nbp && e == cudaSuccess; ++j) {
                const size_t n0 = static_cast<size_t>(j) * bw, wj = n - n0 < bw ? n - n0 : bw;
                e = cudaMemcpy2DAsync(const_cast<double*>(Bd) + n0, ldbs * 8, B + n0, ldb * 8, wj * 8, k,
                                      cudaMemcpyHostToDevice, q->h2d);
                if (e == cudaSuccess)
                    e = cudaEventRecord(q->ev_bp[j], q->h2d);
                if (e == cudaSuccess)
                    e = cudaStreamWaitEvent(q->stream, q->ev_bp[j], 0);
                if (e != cudaSuccess)
                    break;
                st = launch_tiled_dp(q->stream, tile,
                                  make_params(rows, wj, k, alpha, Ad, ldad, Bd + n0, ldbd, beta, Cd + n0, ldcd));
                if (st != KW_OK)
                    break;
            }
            if (st != KW_OK)
                break;
            if (trace)
                cudaEventRecord(tev[1], q->h2d);
        }
        else {
            if (stream_b && pi == 1) {
                // the column-panel uploads of B were waited for on the first stream only
                e = cudaStreamWaitEvent(comp, q->ev_bp[nbp - 1], 0);
                if (e != cudaSuccess)
                    break;
            }
            st = launch_tiled_dp(comp, tile, make_params(rows, n, k, alpha, Ad, ldad, Bd, ldbd, beta, Cd, ldcd));
            if (st != KW_OK)
                break;
        }
        e = cudaGetLastError();
        if (e == cudaSuccess && !c_dev) {
            e = cudaEventRecord(q->ev_ready[s], comp);
            if (e == cudaSuccess)
                e = cudaStreamWaitEvent(q->aux, q->ev_ready[s], 0);
            if (e == cudaSuccess)
                e = cudaMemcpy2DAsync(C + r0 * ldc, ldc * 8, cs, ldcs * 8, n * 8, rows, cudaMemcpyDeviceToHost, q->aux);
            if (e == cudaSuccess)
                e = cudaEventRecord(q->ev_free[s], q->aux);
        }
        else if (e == cudaSuccess) {
            e = cudaEventRecord(q->ev_free[s], comp);
        }
    }
    // A launch that failed part-way still joins what was already enqueued (earlier panels' D2H on
    // the aux stream, the second compute stream) into q->stream before the failure is recorded,
    // so later tasks on the queue cannot overlap it.
    const std::string launch_error = st != KW_OK ? kw::last_error() : std::string();
    const cudaError_t loop_error = e;
    e = cudaSuccess;
    if (trace && loop_error == cudaSuccess && st == KW_OK) {
        cudaEventRecord(tev[2], q->h2d);
        cudaEventRecord(tev[3], (npanels & 1) ? q->stream : q->comp2); // stream of the last panel
        cudaEventRecord(tev[4], q->aux);
    }
    e = cudaEventRecord(q->ev_join, q->aux);
    if (e == cudaSuccess)
        e = cudaStreamWaitEvent(q->stream, q->ev_join, 0);
    if (e == cudaSuccess)
        e = cudaEventRecord(q->ev_join2, q->comp2);
    if (e == cudaSuccess)
        e = cudaStreamWaitEvent(q->stream, q->ev_join2, 0);
    if ((st != KW_OK || loop_error != cudaSuccess) && e == cudaSuccess) {
        // an upload may have been enqueued for a panel that never launched: join it too
        e = cudaEventRecord(q->ev_join, q->h2d);
        if (e == cudaSuccess)
            e = cudaStreamWaitEvent(q->stream, q->ev_join, 0);
    }
    if (st != KW_OK)
        return kw::task_fail(q, "dgemm (host-staged): " + launch_error);
    if (e == cudaSuccess)
        e = loop_error;
    if (trace && e == cudaSuccess) {
        cudaEventSynchronize(tev[4]);
        cudaStreamSynchronize(q->stream);
        float t[5] = {};
        for (int i = 1; i < 5; ++i)
            cudaEventElapsedTime(&t[i], tev[0], tev[i]);
        std::fprintf(stderr, "[kw trace] row panels: %zu x %zu rows | B resident %.2f | last upload %.2f | last compute %.2f | "
                     "last download %.2f ms\n", npanels, R, t[1], t[2], t[3], t[4]);
        for (auto& ev : tev)
            cudaEventDestroy(ev);
    }
    if (e != cudaSuccess)
        return kw::task_fail(q, std::string("dgemm (host-staged): ") + cudaGetErrorString(e));
    return kw::after_enqueue(q, "dgemm");
}

// ------------------------------------------------------------------------------------------
// Streamed e2e DGEMM (all three operands in pinned host memory). The row-panel schedule above
// cannot compute anything useful until the whole of B has crossed PCIe (~10 ms at 8192), and
// every panel launch ends in a partial wave. Here the operands go up in an order that grows
// the computable region as a square — A row panel i, B column panel j, and the C blocks they
// complete — while ONE persistent kernel walks the tiles in that availability order, waiting
// per tile for its panels (ready flags written by the copy stream with cuStreamWriteValue32,
// which fences the copy before the flag). Finished C blocks go back on the aux stream as soon
// as every consumer warp of every tile in the block has counted in (cuStreamWaitValue32 on
// done[block]). Same kernel arithmetic per tile -> bitwise identical to the resident launch.
// k-split (default): the whole schedule first runs over the first quarter of A's columns and
// B's rows (pass 0: k-tiles [0, ktiles/4) of every tile, accumulators parked per thread), then
// over the rest plus C (final pass: reload, remaining k-tiles, epilogue). Square growth unlocks
// s/4 flop per uploaded byte at side s whatever the panel depth, so quarter-depth panels reach
// the kernel's full rate after a quarter of the bytes (DESIGN.md §4 "k-split").
// Deadlock freedom: the kernel waits only on copies, the copies wait only on ev_start (before
// the kernel), the downloads wait on the kernel; everything is enqueued in that order, so even
// streams that share a hardware queue never block a producer behind its consumer.
// ------------------------------------------------------------------------------------------
using PFN_streamValue32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

struct StreamMemOps {
    PFN_streamValue32 write = nullptr, wait = nullptr;
};

const StreamMemOps& stream_mem_ops()
{
    static StreamMemOps ops;
    static std::once_flag once;
    std::call_once(once, [] {
        void* w = nullptr;
        void* t = nullptr;
        cudaDriverEntryPointQueryResult qw, qt;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &w, cudaEnableDefault, &qw) == cudaSuccess &&
            cudaGetDriverEntryPoint("cuStreamWaitValue32", &t, cudaEnableDefault, &qt) == cudaSuccess &&
            qw == cudaDriverEntryPointSuccess && qt == cudaDriverEntryPointSuccess && w && t) {
            ops.write = reinterpret_cast<PFN_streamValue32>(w);
            ops.wait = reinterpret_cast<PFN_streamValue32>(t);
        }
        cudaGetLastError();
    });
    return ops;
}


// Returns KW_OK with *used = false (nothing enqueued) when the streamed schedule does not apply.
kw_status dgemm_streamed(kw::Queue* q, int tile, size_t m, size_t n, size_t k, double alpha, const double* A,
                         size_t lda, const double* B, size_t ldb, double beta, double* C, size_t ldc, bool* used)
{
    KW_NVTX("kw dgemm e2e: streamed");
    *used = false;
    const char* env = std::getenv("KW_E2E_STREAMED");
    if ((env && env[0] == '0') || k == 0 || m > INT_MAX || n > INT_MAX || k > INT_MAX)
        return KW_OK;
    // Only where compute is comparable to the PCIe time: below that the upload is the whole
    // story and the fewer, larger copies of the row-panel schedule win (measured at 4096^3).
    const char* mi = std::getenv("KW_E2E_MIN_INTENSITY");
    const double min_intensity = mi ? std::atof(mi) : 400.0;
    const double intensity = 2.0 * double(m) * double(n) * double(k) /
                             (8.0 * (double(m) * double(k) + double(k) * double(n) + double(m) * double(n)));
    if (intensity < min_intensity)
        return KW_OK;
    const StreamMemOps& ops = stream_mem_ops();
    if (!ops.write || !ops.wait)
        return KW_OK;
    const size_t ldas = round2(k), ldbs = round2(n), ldcs = round2(n);
    // Panel grid: P x P blocks (KW_E2E_PANELS, default 12 — profiles/e2e_dgemm_streamed_r01.txt),
    // edges in whole 128s so both tile shapes nest in every panel.
    const char* pe = std::getenv("KW_E2E_PANELS");
    const long pv = pe ? std::atol(pe) : 0;
    const size_t P = pv > 0 && pv <= 64 ? static_cast<size_t>(pv) : 12;
    const size_t R = std::max<size_t>(128, kw::ceil_div(kw::ceil_div(m, P), 128) * 128);
    const size_t W = std::max<size_t>(128, kw::ceil_div(kw::ceil_div(n, P), 128) * 128);
    const size_t npr = kw::ceil_div(m, R), npc = kw::ceil_div(n, W);
    const int cfg = streamed_config(tile, make_params(m, n, k, alpha, A, lda, B, ldb, beta, C, ldc));
    const StreamedShape shape = streamed_shape(cfg);
    const int bm = shape.bm, bn = shape.bn;
    const uint32_t consumers = shape.consumers;
    const size_t tiles_m = kw::ceil_div(m, bm), tiles_n = kw::ceil_div(n, bn), tiles = tiles_m * tiles_n;
    // k-split (KW_E2E_KSPLIT = d; default 4 from 600 flop/B — 8192^3 is 683 — and off below,
    // where it measured 0.5-1 % slower at 5120-6144; 0/1 = off): a first pass over k-tiles [0, kts), kts =
    // ktiles / d, needs only the first K0 = 16 kts columns of A and rows of B, so d times less
    // upload per unit of work than the full-depth panels — the kernel reaches full rate while
    // most of A and B are still in flight. Its accumulators are parked in `partial` and picked up
    // by the second pass, which streams the rest of A and B and all of C exactly as the
    // single-pass schedule does.
    const size_t ktiles = kw::ceil_div(k, static_cast<size_t>(16));
    const char* ke = std::getenv("KW_E2E_KSPLIT");
    const long kd = ke ? std::atol(ke) : (intensity >= 600.0 ? 4 : 0);
    // Pass boundaries in k-tiles: [0, ktiles/d, ktiles], or KW_E2E_KPASSES = cumulative
    // percentages of the k-tiles ("25,50" -> [0, 25 %, 50 %, 100 %]); empty passes dropped.
    std::vector<size_t> bounds{0};
    if (const char* kp = std::getenv("KW_E2E_KPASSES")) {
        for (const char* c = kp; *c;) {
            char* end = nullptr;
            const long pct = std::strtol(c, &end, 10);
            if (end == c)
                break;
            if (pct > 0 && pct < 100)
                bounds.push_back(ktiles * static_cast<size_t>(pct) / 100);
            c = *end == ',' ? end + 1 : end;
        }
    }
    else if (kd > 1) {
        bounds.push_back(ktiles / static_cast<size_t>(kd));
    }
    bounds.push_back(ktiles);
    std::sort(bounds.begin(), bounds.end());
    bounds.erase(std::unique(bounds.begin(), bounds.end()), bounds.end());
    if (bounds.size() > 16) // the entry's pass index has 4 bits
        bounds.erase(bounds.begin() + 15, bounds.end() - 1);
    const size_t npass = bounds.size() - 1;
    const int passes = static_cast<int>(npass);
    const size_t nflags = npass * (npr + npc) + npr * npc, ndone = npr * npc;
    const size_t mat_bytes = (m * ldas + k * ldbs + m * ldcs) * sizeof(double);
    const size_t part_bytes = passes > 1 ? tiles * bm * bn * sizeof(double) : 0;
    const size_t aux_bytes = (nflags + ndone + 1) * sizeof(uint32_t) + 512; // + the abort word
    if (q->scratch_bytes < mat_bytes + part_bytes + aux_bytes) {
        // growing the scratch: only when the operands fit comfortably (a resource-manager query,
        // so not on every call)
        size_t free_b = 0, total_b = 0;
        if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
            cudaGetLastError();
            return KW_OK;
        }
        if (static_cast<double>(mat_bytes + part_bytes + aux_bytes) >
            0.8 * static_cast<double>(free_b + q->scratch_bytes))
            return KW_OK; // too large to hold whole: the row-panel ring schedule
    }
    kw_status st = kw::ensure_scratch(q, mat_bytes + part_bytes + aux_bytes);
    if (st != KW_OK)
        return st;
    char* base = static_cast<char*>(q->scratch);
    double* Ad = reinterpret_cast<double*>(base);
    double* Bd = Ad + m * ldas;
    double* Cd = Bd + k * ldbs;
    double* part = Cd + m * ldcs; // 16-byte aligned: every extent above is even
    char* tail = reinterpret_cast<char*>(part) + part_bytes;
    tail = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(tail) + 255) & ~uintptr_t(255));
    uint32_t* ready = reinterpret_cast<uint32_t*>(tail);
    uint32_t* done = ready + nflags;

    GemmParams p = make_params(m, n, k, alpha, Ad, ldas, Bd, ldbs, beta, Cd, ldcs);
    if (!tma_eligible(p))
        return KW_OK;
    static std::atomic<int> mem_ops_ok{-1};
    if (mem_ops_ok.load() == 0)
        return KW_OK;
    const size_t grid = static_cast<size_t>(streamed_grid(cfg, p));

    // The growth order: A_0, B_0, then add a B column panel while it is not ahead of the A row
    // panels, else an A row panel; each addition completes the C blocks of its row/column. Every
    // pass follows it with its own k-range of the panels; only the last carries C.
    struct Step {
        bool is_a;
        size_t idx;
    };
    std::vector<Step> steps;
    std::vector<std::pair<size_t, size_t>> blocks; // C blocks in availability order
    {
        size_t a = 0, b = 0;
        while (a < npr || b < npc) {
            const bool add_b = b < npc && (a >= npr || b < a);
            if (add_b) {
                for (size_t i = 0; i < a; ++i)
                    blocks.emplace_back(i, b);
                steps.push_back({false, b++});
            }
            else {
                for (size_t j = 0; j < b; ++j)
                    blocks.emplace_back(a, j);
                steps.push_back({true, a++});
            }
        }
    }
    // Work list: header [0] = {entry count, pass count}, then every pass in the same block order;
    // entry = {tile row, tile col, first k-tile, end k-tile | pass << 27}. Each pass but the last
    // is padded to a multiple of the grid, so a tile's entries all run on one CTA (entry mod grid).
    std::vector<int4> order(1);
    size_t len_last = 0;
    for (size_t ps = 0; ps < npass; ++ps) {
        const int kt0 = static_cast<int>(bounds[ps]), kt1 = static_cast<int>(bounds[ps + 1]);
        const size_t before = order.size();
        for (const auto& bl : blocks) {
            const size_t r0 = bl.first * R, r1 = std::min(m, r0 + R), c0 = bl.second * W, c1 = std::min(n, c0 + W);
            for (size_t tr = r0 / bm; tr < kw::ceil_div(r1, bm); ++tr)
                for (size_t tc = c0 / bn; tc < kw::ceil_div(c1, bn); ++tc)
                    order.push_back(make_int4(static_cast<int>(tr), static_cast<int>(tc), kt0,
                                              kt1 | static_cast<int>(ps << 27)));
        }
        len_last = order.size() - before;
        if (ps + 1 < npass)
            while ((order.size() - 1) % grid != 0)
                order.push_back(make_int4(-1, 0, 0, 0));
    }
    if (len_last != tiles || order.size() > static_cast<size_t>(INT_MAX))
        return kw::task_fail(q, "dgemm (streamed): tile order does not cover the output");
    order[0] = make_int4(static_cast<int>(order.size() - 1), static_cast<int>(npass), 0, 0);

    // The tile order goes up from a pinned copy, once per (scratch, shape, panel grid, tile, passes).
    size_t bhash = 1469598103934665603ull;
    for (size_t b : bounds)
        bhash = (bhash ^ b) * 1099511628211ull;
    const size_t key[8] = {m, n, R, W, static_cast<size_t>(cfg), npass, bhash, grid};
    const bool order_current = std::equal(key, key + 8, q->order_key);
    auto flag = [&](size_t idx) { return reinterpret_cast<CUdeviceptr>(ready + idx); };
    uint32_t* abort_word = done + ndone;
    cudaError_t e = cudaMemsetAsync(ready, 0, (nflags + ndone + 1) * sizeof(uint32_t), q->stream);
    if (e == cudaSuccess && !order_current) {
        if (q->ev_order)
            e = cudaEventSynchronize(q->ev_order); // the previous upload still reads order_host
        else
            e = cudaEventCreateWithFlags(&q->ev_order, cudaEventDisableTiming);
        const size_t bytes = order.size() * sizeof(int4);
        if (e == cudaSuccess && q->order_bytes < bytes) {
            // earlier kernels on this queue may still read order_dev
            e = cudaStreamSynchronize(q->stream);
            if (q->order_host)
                cudaFreeHost(q->order_host);
            if (q->order_dev)
                cudaFree(q->order_dev);
            q->order_host = q->order_dev = nullptr;
            q->order_bytes = 0;
            if (e == cudaSuccess)
                e = cudaHostAlloc(&q->order_host, bytes, cudaHostAllocDefault);
            if (e == cudaSuccess)
                e = cudaMalloc(&q->order_dev, bytes);
            if (e == cudaSuccess)
                q->order_bytes = bytes;
        }
        if (e == cudaSuccess) {
            std::memcpy(q->order_host, order.data(), bytes);
            e = cudaMemcpyAsync(q->order_dev, q->order_host, bytes, cudaMemcpyHostToDevice, q->stream);
        }
        if (e == cudaSuccess)
            e = cudaEventRecord(q->ev_order, q->stream);
        if (e == cudaSuccess)
            std::copy(key, key + 8, q->order_key);
        else
            std::fill(q->order_key, q->order_key + 8, size_t(0));
    }
    if (e == cudaSuccess)
        e = cudaEventRecord(q->ev_start, q->stream);
    if (e == cudaSuccess)
        e = cudaStreamWaitEvent(q->h2d, q->ev_start, 0);
    if (e != cudaSuccess)
        return kw::task_fail(q, std::string("dgemm (streamed): ") + cudaGetErrorString(e));
    if (mem_ops_ok.load() < 0) {
        // Once per process, ordered after the reset above: the stream memory operations must be
        // accepted on this device (a write of the value the reset stored, a wait already
        // satisfied); otherwise nothing but the reset was enqueued and the row-panel schedule runs.
        const bool ok = ops.write(q->h2d, reinterpret_cast<CUdeviceptr>(ready), 0, 0) == CUDA_SUCCESS &&
                        ops.wait(q->h2d, reinterpret_cast<CUdeviceptr>(ready), 0, 0) == CUDA_SUCCESS;
        if (!ok)
            cudaGetLastError();
        mem_ops_ok.store(ok ? 1 : 0);
        if (!ok)
            return KW_OK;
    }
    const bool trace = std::getenv("KW_E2E_TRACE") != nullptr;
    cudaEvent_t tev[5] = {};
    if (trace) {
        for (auto& ev : tev)
            cudaEventCreate(&ev);
        cudaEventRecord(tev[0], q->stream);
    }

    // 1. uploads + ready flags (copy stream): pass by pass, the panels' k-range of A (columns) and
    // B (rows); the last pass also uploads the C blocks each panel completes
    CUresult ce = CUDA_SUCCESS;
    // The C region a step completes: row panel idx x the first `count` column panels (A step) or
    // column panel idx x the first `count` row panels (B step).
    auto upload_c = [&](bool is_a, size_t idx, size_t count) {
        if (is_a) {
            const size_t r0 = idx * R, rows = std::min(m, r0 + R) - r0, cols = std::min(n, count * W);
            e = cudaMemcpy2DAsync(Cd + r0 * ldcs, ldcs * 8, C + r0 * ldc, ldc * 8, cols * 8, rows,
                                  cudaMemcpyHostToDevice, q->h2d);
            for (size_t j = 0; j < count && e == cudaSuccess && ce == CUDA_SUCCESS; ++j)
                ce = ops.write(q->h2d, flag(npass * (npr + npc) + idx * npc + j), 1, 0);
        }
        else {
            const size_t c0 = idx * W, cols = std::min(n, c0 + W) - c0, rows = std::min(m, count * R);
            e = cudaMemcpy2DAsync(Cd + c0, ldcs * 8, C + c0, ldc * 8, cols * 8, rows, cudaMemcpyHostToDevice, q->h2d);
            for (size_t i = 0; i < count && e == cudaSuccess && ce == CUDA_SUCCESS; ++i)
                ce = ops.write(q->h2d, flag(npass * (npr + npc) + i * npc + idx), 1, 0);
        }
    };
    for (size_t ps = 0; ps < npass; ++ps) {
        const bool final_pass = ps + 1 == npass;
        const size_t k0 = bounds[ps] * 16, kw_ = std::min(k, bounds[ps + 1] * 16) - k0;
        const size_t fbase = ps * (npr + npc);
        size_t a = 0, b = 0;
        for (const Step& stp : steps) {
            if (e != cudaSuccess || ce != CUDA_SUCCESS)
                break;
            if (stp.is_a) {
                const size_t r0 = stp.idx * R, rows = std::min(m, r0 + R) - r0;
                e = cudaMemcpy2DAsync(Ad + r0 * ldas + k0, ldas * 8, A + r0 * lda + k0, lda * 8, kw_ * 8, rows,
                                      cudaMemcpyHostToDevice, q->h2d);
                if (e == cudaSuccess)
                    ce = ops.write(q->h2d, flag(fbase + stp.idx), 1, 0);
            }
            else {
                const size_t c0 = stp.idx * W, cols = std::min(n, c0 + W) - c0;
                e = cudaMemcpy2DAsync(Bd + k0 * ldbs + c0, ldbs * 8, B + k0 * ldb + c0, ldb * 8, cols * 8, kw_,
                                      cudaMemcpyHostToDevice, q->h2d);
                if (e == cudaSuccess)
                    ce = ops.write(q->h2d, flag(fbase + npr + stp.idx), 1, 0);
            }
            const size_t count = stp.is_a ? b : a; // blocks this step completes
            if (stp.is_a)
                ++a;
            else
                ++b;
            // the final pass's C blocks go up right behind the panel that completes them (one step
            // later measured 0.6 % slower at 8192^3, neutral elsewhere)
            if (final_pass && count > 0 && e == cudaSuccess && ce == CUDA_SUCCESS)
                upload_c(stp.is_a, stp.idx, count);
        }
    }
    if (e != cudaSuccess || ce != CUDA_SUCCESS)
        return kw::task_fail(q, "dgemm (streamed): upload schedule failed");
    *used = true;
    if (trace)
        cudaEventRecord(tev[3], q->h2d);
    if (trace)
        cudaEventRecord(tev[1], q->stream);

    // 2. the persistent kernel (queue stream)
    p.tile_list = static_cast<const int4*>(q->order_dev);
    p.ready = ready; // done[] follows the flags (GemmParams)
    p.partial = part;
    p.panel_rows = static_cast<int>(R);
    p.panel_cols = static_cast<int>(W);
    p.npr = static_cast<int>(npr);
    p.npc = static_cast<int>(npc);
    st = launch_streamed(q->stream, cfg, p);
    if (st != KW_OK)
        return kw::task_fail(q, kw::last_error());
    e = cudaGetLastError();
    // The kernel's abort word -> this task's failure slot (resolved by kw_queue_wait).
    if (auto fs = kw::make_slot("dgemm (streamed)")) {
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(fs->slot, abort_word, sizeof(uint32_t), cudaMemcpyDeviceToHost, q->stream);
        if (e == cudaSuccess)
            kw::arm_slot(q, std::move(fs));
        else
            kw::release_slot(*fs);
    }
    if (trace)
        cudaEventRecord(tev[2], q->stream);

    // 3. downloads, block by block as they complete (aux stream)
    if (e == cudaSuccess)
        e = cudaStreamWaitEvent(q->aux, q->ev_start, 0);
    for (size_t bi = 0; bi < blocks.size() && e == cudaSuccess && ce == CUDA_SUCCESS; ++bi) {
        const size_t i = blocks[bi].first, j = blocks[bi].second;
        const size_t r0 = i * R, rows = std::min(m, r0 + R) - r0, c0 = j * W, cols = std::min(n, c0 + W) - c0;
        const uint32_t expect = static_cast<uint32_t>(kw::ceil_div(rows, bm) * kw::ceil_div(cols, bn)) * consumers;
        ce = ops.wait(q->aux, reinterpret_cast<CUdeviceptr>(done + i * npc + j), expect, 0 /* GEQ */);
        if (ce == CUDA_SUCCESS)
            e = cudaMemcpy2DAsync(C + r0 * ldc + c0, ldc * 8, Cd + r0 * ldcs + c0, ldcs * 8, cols * 8, rows,
                                  cudaMemcpyDeviceToHost, q->aux);
    }
    if (e == cudaSuccess && ce == CUDA_SUCCESS) {
        e = cudaEventRecord(q->ev_join, q->aux);
        if (e == cudaSuccess)
            e = cudaStreamWaitEvent(q->stream, q->ev_join, 0);
    }
    if (e != cudaSuccess || ce != CUDA_SUCCESS)
        return kw::task_fail(q, "dgemm (streamed): download schedule failed");
    if (trace) {
        cudaEventRecord(tev[4], q->aux);
        cudaEventSynchronize(tev[4]);
        cudaStreamSynchronize(q->stream);
        float t[5] = {};
        for (int i = 1; i < 5; ++i)
            cudaEventElapsedTime(&t[i], tev[0], tev[i]);
        std::fprintf(stderr, "[kw trace] kernel start %.2f end %.2f | last upload %.2f | last download %.2f ms\n",
                     t[1], t[2], t[3], t[4]);
        for (auto& ev : tev)
            cudaEventDestroy(ev);
    }
    return kw::after_enqueue(q, "dgemm");
}


} // namespace kw::gemm
