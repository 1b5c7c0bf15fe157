// kw_dgemm.cu — K2 tiled DGEMM (FP64 DMMA tensor cores) and K3 naive bit-exact DGEMM, sm_100a.
//
// Reference: GemmTiledKernel (/root/reference/proj/core/src/kernels/gemm.cpp:40-118),
// GemmNaiveKernel (gemm.cpp:11-38), gemmReference oracle (core/src/kernels/reference.cpp:14-26).
//
// K2 design (FP64 on Blackwell): tcgen05.mma has no f64 kind, so FP64 tensor work is the legacy
// DMMA.8x8x4 (mma.sync.m8n8k4.f64). Measured on this pool's B200: DMMA 37.2 TFLOP/s vs DFMA
// 34.1 TFLOP/s peak (tools/probe/probe.cu), and DMMA needs 8x fewer operand registers per FMA.
//   * primary kernel dgemm_tma_kernel: warp-specialised — one producer lane streams k-tiles of
//     A and B with TMA (cp.async.bulk.tensor, SWIZZLE_128B, hardware zero-fill of ragged edges)
//     into an mbarrier-synchronised stage ring; consumer warps (64 x 32 warp tiles = 8 x 4 DMMA
//     accumulators) wait `full`, run the DMMAs, release `empty` once the DMMAs of the stage's last
//     k-step are issued (not earlier: a pending LDS must not race the refill's TMA); no CTA
//     barrier in the main loop;
//     setmaxnreg moves registers from the producer warpgroup to the consumers;
//   * a paired k-slot permutation puts two k-steps of an A fragment in one 16-byte chunk (one
//     LDS.128), conflict-free under the swizzle; every tile shape ("paired" configs 14-17) feeds
//     each output element the identical DMMA sequence, so the per-problem tile choice
//     (pick_config: 64 x 128 at 2 CTAs/SM or 64 x 64 at 3) never changes a bit;
//   * epilogue fl(fl(alpha*acc) + fl(beta*c)) exactly as gemm.cpp:115 / reference.cpp:24 (C is
//     always read, also for beta == 0); tiles rasterised in groups of 8 tile-rows for L2 reuse;
//   * the STREAMED instantiation additionally walks a tile list and waits on per-panel ready
//     flags (host-operand e2e path, kw_dgemm_e2e.cu); list entries carry a k-tile range, so a
//     tile can run as two passes whose accumulators are parked in global memory in between;
//   * dgemm_dmma_kernel: the earlier cp.async (LDGSTS) + __syncthreads family, kept as the path
//     for operands TMA cannot address (odd leading dimensions) and for the tile sweep.
// Numerics: per output element the K products are accumulated in ascending k-tile order by
// DMMA (fused multiply-add), hence |dC| <= (K+4)*2^-53*|C_ref| instead of bit equality
// (SURVEY.md §7 "Hard parts" 6). K3 (naive) and K2-bitwise below are the bit-exact modes.
#include "kw_common.cuh"
#include "kw_dgemm_internal.cuh"

#include <cuda.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <utility>
#include <vector>

namespace {

// ------------------------------------------------------------------------------------------
// PTX helpers
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes));
}

__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src, int src_bytes)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes));
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

template <int N>
__device__ __forceinline__ void cp_async_wait()
{
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// D += A(8x4, row) * B(4x8, col), fp64. Lane (g = lane/4, t = lane%4) supplies A[g][t] and
// B[t][g] and owns D[g][2t], D[g][2t+1].
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b)
{
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}

// ------------------------------------------------------------------------------------------
// K2: DMMA tiled kernel
// ------------------------------------------------------------------------------------------
template <int BM_, int BN_, int BK_, int WM_, int WN_, int STAGES_, int MIN_BLOCKS_ = 1>
struct TileCfg {
    static constexpr int BM = BM_, BN = BN_, BK = BK_, WM = WM_, WN = WN_, STAGES = STAGES_;
    static constexpr int MIN_BLOCKS = MIN_BLOCKS_;
    static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
    static constexpr int THREADS = 32 * WARPS_M * WARPS_N;
    static constexpr int MT = WM / 8, NT = WN / 8; // DMMA tiles per warp
    static constexpr int A_STAGE = BM * BK, B_STAGE = BK * BN; // doubles
    static constexpr size_t SMEM = static_cast<size_t>(STAGES) * (A_STAGE + B_STAGE) * sizeof(double);
    static_assert(BK == 16 || BK == 32, "A swizzle assumes >= 8 16-byte chunks per A row");
    static_assert(BN % 16 == 0 && BM % 8 == 0, "tile shape");
    static_assert((BM * BK / 2) % THREADS == 0 && (BK * BN / 2) % THREADS == 0, "load split");
};

// Element offsets (in doubles) inside one stage.
template <int BK>
__device__ __forceinline__ int a_off(int m, int k)
{
    return m * BK + ((((k >> 1) ^ ((m & 3) << 1))) << 1) + (k & 1);
}
template <int BN>
__device__ __forceinline__ int b_off(int k, int n)
{
    return k * BN + ((((n >> 1) ^ ((k & 3) << 1))) << 1) + (n & 1);
}

using kw::gemm::GemmParams;

// Dynamic shared memory above 48 KiB is opted into per kernel AND per device: a process that
// drives several GPUs must set the attribute on each of them.
kw_status ensure_smem(const void* fn, size_t bytes, const char* what)
{
    int dev = 0;
    cudaGetDevice(&dev);
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    std::lock_guard<std::mutex> lock(mu);
    if (done.count({fn, dev}))
        return KW_OK;
    const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
    if (e != cudaSuccess)
        return kw::cuda_fail(what, e);
    done.insert({fn, dev});
    return KW_OK;
}

template <class Cfg, bool VEC16>
__device__ __forceinline__ void load_stage(const GemmParams& p, double* sA, double* sB, int bm, int bn, int k0,
                                           int tid)
{
    // A tile: BM rows x BK cols = BM * (BK/2) chunks of two doubles.
    constexpr int A_CHUNKS = Cfg::BM * Cfg::BK / 2;
#pragma unroll
    for (int i = 0; i < A_CHUNKS / Cfg::THREADS; ++i) {
        const int c = tid + i * Cfg::THREADS;
        const int row = c / (Cfg::BK / 2), kc = c % (Cfg::BK / 2);
        const int gm = bm + row, gk = k0 + kc * 2;
        int valid = 0;
        if (gm < p.m) {
            valid = p.k - gk;
            valid = valid < 0 ? 0 : (valid > 2 ? 2 : valid);
        }
        const double* src = valid > 0 ? p.a + gm * p.lda + gk : p.a;
        const uint32_t dst = smem_u32(sA + a_off<Cfg::BK>(row, kc * 2));
        if (VEC16) {
            cp_async16(dst, src, valid * 8);
        }
        else {
            cp_async8(dst, src, valid >= 1 ? 8 : 0);
            cp_async8(dst + 8, valid >= 2 ? src + 1 : p.a, valid >= 2 ? 8 : 0);
        }
    }
    // B tile: BK rows x BN cols.
    constexpr int B_CHUNKS = Cfg::BK * Cfg::BN / 2;
#pragma unroll
    for (int i = 0; i < B_CHUNKS / Cfg::THREADS; ++i) {
        const int c = tid + i * Cfg::THREADS;
        const int row = c / (Cfg::BN / 2), nc = c % (Cfg::BN / 2);
        const int gk = k0 + row, gn = bn + nc * 2;
        int valid = 0;
        if (gk < p.k) {
            valid = p.n - gn;
            valid = valid < 0 ? 0 : (valid > 2 ? 2 : valid);
        }
        const double* src = valid > 0 ? p.b + gk * p.ldb + gn : p.b;
        const uint32_t dst = smem_u32(sB + b_off<Cfg::BN>(row, nc * 2));
        if (VEC16) {
            cp_async16(dst, src, valid * 8);
        }
        else {
            cp_async8(dst, src, valid >= 1 ? 8 : 0);
            cp_async8(dst + 8, valid >= 2 ? src + 1 : p.b, valid >= 2 ? 8 : 0);
        }
    }
}

template <class Cfg, bool VEC16>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MIN_BLOCKS) dgemm_dmma_kernel(GemmParams p)
{
    extern __shared__ __align__(128) double smem[];
    double* sA = smem;
    double* sB = smem + Cfg::STAGES * Cfg::A_STAGE;

    // Grouped rasterisation: runs of 8 tile-rows sweep the tile-columns together.
    constexpr int GROUP = 8;
    const int tile = blockIdx.x;
    const int per_group = GROUP * p.tiles_n;
    const int group = tile / per_group;
    const int first_m = group * GROUP;
    const int gsize = (p.tiles_m - first_m) < GROUP ? (p.tiles_m - first_m) : GROUP;
    const int in_group = tile - group * per_group;
    const int tm = first_m + in_group % gsize;
    const int tn = in_group / gsize;
    const int bm = tm * Cfg::BM, bn = tn * Cfg::BN;

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int wm = (warp / Cfg::WARPS_N) * Cfg::WM;
    const int wn = (warp % Cfg::WARPS_N) * Cfg::WN;
    const int g = lane >> 2, t = lane & 3;

    double acc[Cfg::MT][Cfg::NT][2];
#pragma unroll
    for (int i = 0; i < Cfg::MT; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::NT; ++j)
            acc[i][j][0] = acc[i][j][1] = 0.0;

    const int ktiles = (p.k + Cfg::BK - 1) / Cfg::BK;
#pragma unroll
    for (int s = 0; s < Cfg::STAGES - 1; ++s) {
        if (s < ktiles)
            load_stage<Cfg, VEC16>(p, sA + s * Cfg::A_STAGE, sB + s * Cfg::B_STAGE, bm, bn, s * Cfg::BK, tid);
        cp_async_commit();
    }

    for (int kt = 0; kt < ktiles; ++kt) {
        cp_async_wait<Cfg::STAGES - 2>();
        __syncthreads();
        {
            const int nk = kt + Cfg::STAGES - 1;
            if (nk < ktiles) {
                const int s = nk % Cfg::STAGES;
                load_stage<Cfg, VEC16>(p, sA + s * Cfg::A_STAGE, sB + s * Cfg::B_STAGE, bm, bn, nk * Cfg::BK, tid);
            }
            cp_async_commit();
        }
        const int s = kt % Cfg::STAGES;
        const double* a_s = sA + s * Cfg::A_STAGE;
        const double* b_s = sB + s * Cfg::B_STAGE;
#pragma unroll
        for (int kk = 0; kk < Cfg::BK / 4; ++kk) {
            double af[Cfg::MT], bf[Cfg::NT];
            const int k = kk * 4 + t;
#pragma unroll
            for (int i = 0; i < Cfg::MT; ++i)
                af[i] = a_s[a_off<Cfg::BK>(wm + i * 8 + g, k)];
#pragma unroll
            for (int j = 0; j < Cfg::NT; ++j)
                bf[j] = b_s[b_off<Cfg::BN>(k, wn + j * 8 + g)];
#pragma unroll
            for (int i = 0; i < Cfg::MT; ++i)
#pragma unroll
                for (int j = 0; j < Cfg::NT; ++j)
                    dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
    }
    cp_async_wait<0>();

    // Epilogue: C = fl(fl(alpha*acc) + fl(beta*c)).
    const bool c_vec = (p.ldc % 2 == 0) && (reinterpret_cast<uintptr_t>(p.c) % 16 == 0);
#pragma unroll
    for (int i = 0; i < Cfg::MT; ++i) {
        const int row = bm + wm + i * 8 + g;
        if (row >= p.m)
            continue;
        double* crow = p.c + row * p.ldc;
#pragma unroll
        for (int j = 0; j < Cfg::NT; ++j) {
            const int col = bn + wn + j * 8 + 2 * t;
            if (c_vec && col + 1 < p.n) {
                double2 old = *reinterpret_cast<const double2*>(crow + col);
                double2 out;
                out.x = __dadd_rn(__dmul_rn(p.alpha, acc[i][j][0]), __dmul_rn(p.beta, old.x));
                out.y = __dadd_rn(__dmul_rn(p.alpha, acc[i][j][1]), __dmul_rn(p.beta, old.y));
                *reinterpret_cast<double2*>(crow + col) = out;
            }
            else {
                if (col < p.n)
                    crow[col] = __dadd_rn(__dmul_rn(p.alpha, acc[i][j][0]), __dmul_rn(p.beta, crow[col]));
                if (col + 1 < p.n)
                    crow[col + 1] = __dadd_rn(__dmul_rn(p.alpha, acc[i][j][1]), __dmul_rn(p.beta, crow[col + 1]));
            }
        }
    }
}


// ------------------------------------------------------------------------------------------
// K2 (primary): warp-specialised TMA + mbarrier DMMA kernel.
//   * one producer warp: a single elected lane streams k-tiles of A (box 16 x BM) and B
//     (BN/16 boxes of 16 x 16) into a STAGES-deep shared ring with cp.async.bulk.tensor
//     (TMA, SWIZZLE_128B, hardware zero-fill of ragged edges), signalling `full[s]` through
//     the transaction count; it waits on `empty[s]` before reusing a slot;
//   * CONSUMERS DMMA warps: wait `full[s]`, run the 4 k-steps of the tile, arrive on
//     `empty[s]` — no CTA-wide barrier anywhere in the main loop, so warps drift freely and
//     fill each other's issue gaps;
//   * k-slot permutation: DMMA step s of a k-tile feeds lane t with
//         k(s, t) = 8*(t>>1) + 2*((t+s)&3) + (t&1)
//     (the 4 steps still cover the 16 k of the tile exactly once). Under the 128-byte TMA
//     swizzle this makes every LDS.64 fragment load of A and of B hit 16 distinct banks per
//     half-warp (proof in DESIGN.md §K2). Only the grouping of products inside a DMMA changes,
//     which is within the stated (K+4)u tolerance and identical for every output element.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE_%=;\n"
        "bra WAIT_%=;\n"
        "DONE_%=:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map)
{
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* flag)
{
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(flag) : "memory");
    return v;
}

// Streamed mode: waits until the copy stream has published a panel (ready flag != 0). Bounded,
// and never a trap (a trap would poison the CUDA context for every queue in the process): a flag
// that has not arrived after ~2^26 polls sets the launch's abort word (the launcher copies it
// into the task's failure slot, so kw_queue_wait reports KW_FAIL_READY_TIMEOUT) and returns; once
// the abort word is set every later wait returns at once, so the kernel drains quickly instead
// of hanging the GPU, with the task already failed.
__device__ __forceinline__ void wait_ready(const uint32_t* flag, uint32_t* abort)
{
    uint32_t ns = 64;
    for (long long spins = 0;; ++spins) {
        if (ld_acquire_gpu(flag) != 0)
            return;
        if ((spins & 255) == 0 && *reinterpret_cast<volatile uint32_t*>(abort) != 0)
            return;
        if (spins > (1ll << 26)) {
            atomicExch(abort, KW_FAIL_READY_TIMEOUT);
            return;
        }
        __nanosleep(ns);
        ns = ns < 2048 ? ns * 2 : ns;
    }
}

#ifndef KW_DGEMM_REG_PREFETCH_C
#define KW_DGEMM_REG_PREFETCH_C 1 // 1-CTA/SM SPLIT tiles: C read into registers at tile start
#endif
#ifndef KW_DGEMM_C_L2PF
#define KW_DGEMM_C_L2PF 1 // L2 prefetch of the C block at tile start (A/B: -DKW_DGEMM_C_L2PF=0)
#endif
#ifndef KW_DGEMM_AHEAD2
#define KW_DGEMM_AHEAD2 1 // two-step fragment prefetch for small warp tiles (A/B: -DKW_DGEMM_AHEAD2=0)
#endif
template <int BM_, int BN_, int WM_, int WN_, int STAGES_, int MIN_BLOCKS_ = 1, bool PAIRED_ = false,
          int GROUPS_ = 1>
struct TmaCfg {
    static constexpr int BM = BM_, BN = BN_, BK = 16, WM = WM_, WN = WN_, STAGES = STAGES_;
    // PAIRED: k-slot map k = 8(t>>1) + 4(t&1) + 2((t>>1)^(s>>1)) + (s&1) puts the A fragments
    // of k-steps 2q and 2q+1 in one 16-byte chunk -> A via LDS.128 (still conflict-free).
    static constexpr bool PAIRED = PAIRED_;
    static constexpr int MIN_BLOCKS = MIN_BLOCKS_; // co-resident CTAs per SM
    static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
    static constexpr int CONSUMERS = WARPS_M * WARPS_N; // per consumer group
    // GROUPS > 1: that many independent consumer groups in one CTA, each with its own stage ring,
    // producer lane and tile sequence (virtual CTAs sharing one SM's registers and one producer
    // warpgroup — see the SPLIT notes).
    static constexpr int GROUPS = GROUPS_;
    static constexpr int TOTAL_CONSUMERS = CONSUMERS * GROUPS;
    // Consumer warps + one producer warpgroup (4 warps: one issues TMA per group, the others exit).
    // setmaxnreg moves registers from the producer warpgroup to the consumers.
    static constexpr int THREADS = 32 * (TOTAL_CONSUMERS + 4);
    static constexpr int PRODUCER_REGS = 40;
    // The CTA's register pool is fixed at launch: ptxas pins a setmaxnreg kernel to the
    // launch-bounds cap, floor(65536 / roundup(THREADS, 128) / 8) * 8 per thread. setmaxnreg.inc
    // blocks until registers are free, so the consumers may only take what the producer
    // warpgroup releases — asking for more deadlocks the CTA.
    static constexpr int LAUNCH_REGS_RAW = (65536 / MIN_BLOCKS / (((THREADS + 127) / 128) * 128)) / 8 * 8;
    static constexpr int LAUNCH_REGS = LAUNCH_REGS_RAW > 255 ? 255 : LAUNCH_REGS_RAW;
    static constexpr int POOL_PER_LANE = LAUNCH_REGS * (TOTAL_CONSUMERS + 4);
    static constexpr int CONSUMER_REGS_RAW = ((POOL_PER_LANE - 4 * PRODUCER_REGS) / TOTAL_CONSUMERS) / 8 * 8;
    static constexpr int CONSUMER_REGS = CONSUMER_REGS_RAW > 240 ? 240 : CONSUMER_REGS_RAW;
    // Small CTAs already get (nearly) 255 registers per thread: no redistribution needed.
    static constexpr bool REBALANCE = CONSUMER_REGS > LAUNCH_REGS;
    static_assert(4 * PRODUCER_REGS + TOTAL_CONSUMERS * CONSUMER_REGS <= POOL_PER_LANE, "register pool overcommitted");
    static_assert(TOTAL_CONSUMERS % 4 == 0, "consumer warps form whole warpgroups (setmaxnreg granularity)");
    static_assert(GROUPS >= 1 && GROUPS <= 4, "one producer warp per consumer group");
    static constexpr int MT = WM / 8, NT = WN / 8;
    static constexpr uint32_t A_BYTES = BM * 128; // BM rows of 16 doubles
    static constexpr uint32_t B_BYTES = BN * 128; // BN/16 boxes of 16 x 16 doubles (2 KB)
    static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr size_t SMEM =
        1024 + static_cast<size_t>(GROUPS) * STAGES * STAGE_BYTES + 2 * GROUPS * STAGES * sizeof(uint64_t);
    static_assert(WN % 16 == 0 && BN % 16 == 0 && BM <= 256, "tile shape");
};

// SPLIT (resident operands, one persistent CTA per SM): the T x K k-tiles of the problem
// (T output tiles, K k-tiles each) are cut into G equal contiguous ranges in (tile, k-tile)
// order, one per CTA, so every SM gets the same number of k-tiles however T divides by G (the
// wave-quantisation loss of small outputs: 256 tiles on 148 SMs). A tile that straddles two
// ranges runs as a head piece [0, x) on CTA c and a tail piece [x, K) on CTA c + 1: the head
// parks its accumulators (exact doubles) in slot c and raises a per-warp flag; the tail waits
// for the flag, reloads them and continues the same DMMA chain — same thread role, same k
// order, so the bits equal a one-CTA tile (no split-k reduction; the bits do not depend on M,
// N, G or the piece boundaries). Each CTA runs its head piece FIRST and its tail piece LAST,
// and CTA indices are taken from an atomic ticket in start order, so the CTA a tail waits on
// is already running and its head piece depends on nothing: no wait can deadlock.
// Scratch (per stream, kw::gemm::split_scratch): p.ready = [u64 ticket][u64 abort-word pointer]
// [G * CONSUMERS u32 flags], p.partial = G park slots of CONSUMERS * MT * NT * 32 double2.
struct SplitRange {
    int ndp, dp0, dp_step;     // data-parallel tiles dp0 + j * dp_step, j < ndp (run first)
    int head, nfull, tail;     // piece counts (head/tail 0 or 1)
    int t_head, x_head;        // head piece: tile, k-tiles [0, x_head)
    int t_full0;               // first full tile
    int t_tail, x_tail;        // tail piece: tile, k-tiles [x_tail, K)
};
// Tiles [0, Tdp) run data-parallel (CTA c: tiles c, c + G, ...: concurrent CTAs work on
// neighbouring tiles, the L2 locality of the ordinary grid); the last Ts = T - Tdp tiles
// (G <= Ts < 2G by default) are cut into the equal k-tile ranges. dp_override >= 0 sets Tdp.
__host__ __device__ inline long long split_dp_tiles(long long T, long long G, long long dp_override)
{
    const long long cap = T >= G ? (T - G) / G * G : 0; // leaves >= G tiles to the ranges
    if (dp_override >= 0)
        return dp_override / G * G < cap ? dp_override / G * G : cap;
    return cap;
}
__host__ __device__ inline SplitRange split_range(long long T, long long K, long long G, long long c,
                                                   long long dp_override = -1)
{
    SplitRange r{};
    const long long Tdp = split_dp_tiles(T, G, dp_override);
    r.ndp = static_cast<int>(Tdp / G);
    r.dp0 = static_cast<int>(c);
    r.dp_step = static_cast<int>(G);
    const long long W = (T - Tdp) * K, lo = Tdp * K + W * c / G, hi = Tdp * K + W * (c + 1) / G;
    if (hi <= lo)
        return r;
    const long long tf = lo / K, tl = (hi - 1) / K;
    r.tail = (lo % K) != 0;
    r.t_tail = static_cast<int>(tf);
    r.x_tail = static_cast<int>(lo % K);
    r.head = (hi % K) != 0 && tl > tf;
    r.t_head = static_cast<int>(tl);
    r.x_head = static_cast<int>(hi % K);
    const long long f0 = r.tail ? tf + 1 : tf, f1 = (hi % K) != 0 ? tl : tl + 1; // full tiles [f0, f1)
    r.t_full0 = static_cast<int>(f0);
    r.nfull = f1 > f0 ? static_cast<int>(f1 - f0) : 0;
    return r;
}

// Reports a piece wait that timed out (abort word, see kw_queue_wait) instead of hanging the GPU.
__device__ __noinline__ void split_abort(const uint32_t* scratch, int lane)
{
    uint32_t* abort = *reinterpret_cast<uint32_t* const*>(scratch + 2);
    if (lane == 0 && abort)
        atomicExch_system(abort, KW_FAIL_READY_TIMEOUT);
}

// KRANGE: a data-parallel launch over one k-tile range [p.npr, p.npc) of every tile — accumulators
// reloaded from (kt0 > 0) and parked to (kt1 < K) p.partial per tile, so a product can run as
// several launches in k order with the bits of one launch (the row-sharded DGEMM's k-slab
// passes: each pass only needs the B rows broadcast so far).
template <class Cfg, bool STREAMED = false, bool SPLIT = false, bool KRANGE = false>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MIN_BLOCKS)
    dgemm_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmParams p)
{
    static_assert(int(STREAMED) + int(SPLIT) + int(KRANGE) <= 1, "one tile-walk mode");
    static_assert(!KRANGE || Cfg::GROUPS == 1, "k-range launches use one consumer group");
    static_assert(!STREAMED || Cfg::GROUPS == 1, "streamed launches use one consumer group");
    extern __shared__ uint8_t smem_raw[];
    // 1 KiB alignment (128B-swizzled TMA boxes) by pointer arithmetic on the __shared__ array, not
    // through an integer cast: the compiler must still see a shared-space pointer, so fragment
    // loads compile to LDS. (Through uintptr_t they became generic LD.E — slower, and not ordered
    // before the empty-barrier arrive, so a refill could overwrite a stage still being read.)
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* full_all = reinterpret_cast<uint64_t*>(smem + Cfg::GROUPS * Cfg::STAGES * Cfg::STAGE_BYTES);
    uint64_t* empty_all = full_all + Cfg::GROUPS * Cfg::STAGES;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    // consumer group of this warp (producer warp TOTAL_CONSUMERS + g serves group g)
    const int grp = Cfg::GROUPS == 1 ? 0 // a compile-time 0 keeps the one-group kernels' codegen
                    : warp < Cfg::TOTAL_CONSUMERS ? warp / Cfg::CONSUMERS
                    : (warp - Cfg::TOTAL_CONSUMERS < Cfg::GROUPS ? warp - Cfg::TOTAL_CONSUMERS : 0);
    uint8_t* const ring = smem + grp * Cfg::STAGES * Cfg::STAGE_BYTES; // this group's stage ring
    uint64_t* const full = full_all + grp * Cfg::STAGES;
    uint64_t* const empty = empty_all + grp * Cfg::STAGES;

    // Grouped rasterisation: runs of 8 tile-rows sweep the tile-columns together. A CTA walks
    // tiles blockIdx.x, +gridDim.x, ... (one tile when the grid covers every tile; a persistent
    // grid keeps the smem ring running across tiles, so the producer fills the next tile's
    // stages while the consumers run the epilogue). All CTAs at step j work on consecutive tile
    // ids, which keeps the L2 locality of the rasterisation.
    // tile-rows per raster group (resident launches: p.panel_rows when > 1, see dgemm_group())
    const int GROUP = (!STREAMED && p.panel_rows > 1) ? p.panel_rows : 8;
    int ntiles = STREAMED ? p.tile_list[0].x : p.tiles_m * p.tiles_n;
    const int ktiles = (p.k + Cfg::BK - 1) / Cfg::BK;
    // SPLIT: this CTA's plan lives in shared memory (read per piece) — per-thread copies cost the
    // 2- and 3-CTA/SM configurations their register budget (spills).
    __shared__ SplitRange sr_all[Cfg::GROUPS];
    SplitRange& sr = sr_all[grp];
    // Tile origin and k-tile range [kt0, kt1) of work item `tile`; false = padding entry.
    auto origin = [&](int tile, int& bm, int& bn, int& kt0, int& kt1) {
        if constexpr (STREAMED) {
            const int4 v = p.tile_list[1 + tile];
            bm = v.x * Cfg::BM;
            bn = v.y * Cfg::BN;
            kt0 = v.z;
            kt1 = v.w & 0x07ffffff; // bits 27..30: the entry's pass (its set of panel flags)
            return v.x >= 0;
        }
        if constexpr (SPLIT) {
            // piece `tile` of this CTA: data-parallel tiles, then head, full tiles, tail
            if (tile < sr.ndp) {
                kt0 = 0;
                kt1 = ktiles;
                tile = sr.dp0 + tile * sr.dp_step;
            }
            else if ((tile -= sr.ndp) < sr.head) {
                kt0 = 0;
                kt1 = sr.x_head;
                tile = sr.t_head;
            }
            else if (tile < sr.head + sr.nfull) {
                kt0 = 0;
                kt1 = ktiles;
                tile = sr.t_full0 + (tile - sr.head);
            }
            else {
                kt0 = sr.x_tail;
                kt1 = ktiles;
                tile = sr.t_tail;
            }
        }
        else if constexpr (KRANGE) {
            if (p.panel_cols > 0) { // split-k: slice blockIdx.y of p.panel_cols k-tiles
                kt0 = static_cast<int>(blockIdx.y) * p.panel_cols;
                kt1 = kt0 + p.panel_cols < ktiles ? kt0 + p.panel_cols : ktiles;
            }
            else {
                kt0 = p.npr;
                kt1 = p.npc;
            }
        }
        else {
            kt0 = 0;
            kt1 = ktiles;
        }
        const int per_group = GROUP * p.tiles_n;
        const int group = tile / per_group;
        const int first_m = group * GROUP;
        const int gsize = (p.tiles_m - first_m) < GROUP ? (p.tiles_m - first_m) : GROUP;
        const int in_group = tile - group * per_group;
        bm = (first_m + in_group % gsize) * Cfg::BM;
        bn = (in_group / gsize) * Cfg::BN;
        return true;
    };

    if (tid == 0) {
        for (int s = 0; s < Cfg::GROUPS * Cfg::STAGES; ++s) {
            mbar_init(&full_all[s], 1);
            mbar_init(&empty_all[s], Cfg::CONSUMERS);
        }
        fence_mbar_init();
    }
    // Programmatic dependent launch: the next grid on the stream may start its launch and the
    // barrier setup above while this one drains; nothing in global memory (A, B, C, the split
    // scratch) is touched before the previous grid has completed.
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    // SPLIT: this CTA's range index = its start-order ticket (see split_range)
    // Virtual CTAs: consumer group g of CTA b is virtual CTA b * GROUPS + g of gridDim.x * GROUPS.
    int first = blockIdx.x * Cfg::GROUPS + grp, step = gridDim.x * Cfg::GROUPS, ticket = 0;
    if constexpr (SPLIT) {
        __shared__ int s_ticket;
        if (tid == 0) {
            const int tk = static_cast<int>(atomicAdd(reinterpret_cast<unsigned long long*>(p.ready), 1ull) % gridDim.x);
            s_ticket = tk;
            for (int g2 = 0; g2 < Cfg::GROUPS; ++g2)
                sr_all[g2] = split_range(static_cast<long long>(p.tiles_m) * p.tiles_n, ktiles,
                                         static_cast<long long>(gridDim.x) * Cfg::GROUPS, tk * Cfg::GROUPS + g2, p.npr);
        }
        __syncthreads();
        ticket = s_ticket * Cfg::GROUPS + grp; // this group's virtual ticket
        ntiles = sr.ndp + sr.head + sr.nfull + sr.tail;
        first = 0;
        step = 1;
    }
    else {
        __syncthreads();
    }

    // SPLIT gives its producer warpgroup the minimum (24: one lane issues TMA from a short plan)
    // so the consumers keep the registers the split bookkeeping costs (2- and 3-CTA/SM tiles
    // spilled with 40).
    constexpr int PREGS = (SPLIT && Cfg::MIN_BLOCKS > 1) ? 24 : Cfg::PRODUCER_REGS;
    constexpr int CREGS_RAW = ((Cfg::POOL_PER_LANE - 4 * PREGS) / Cfg::TOTAL_CONSUMERS) / 8 * 8;
    constexpr int CREGS = CREGS_RAW > 240 ? 240 : CREGS_RAW;
    static_assert(4 * PREGS + Cfg::TOTAL_CONSUMERS * CREGS <= Cfg::POOL_PER_LANE, "register pool overcommitted");
    if (warp >= Cfg::TOTAL_CONSUMERS) {
        // ---------------- producer warpgroup ----------------
        if constexpr (Cfg::REBALANCE)
            asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(PREGS));
        if (warp - Cfg::TOTAL_CONSUMERS < Cfg::GROUPS && lane == 0) {
            tma_prefetch_desc(&tmA);
            tma_prefetch_desc(&tmB);
            int it = 0; // k-tile iteration counter across this CTA's tiles (ring position)
            // streamed: the abort word follows the done[] counters (GemmParams)
            uint32_t* abort = nullptr;
            if constexpr (STREAMED)
                abort = p.ready + p.tile_list[0].y * (p.npr + p.npc) + 2 * p.npr * p.npc;
            for (int tile = first; tile < ntiles; tile += step) {
                int bm, bn, kt0, kt1;
                if (!origin(tile, bm, bn, kt0, kt1))
                    continue;
                if constexpr (STREAMED) {
                    // A row panel and B column panel of this tile (of its pass) resident? (The C
                    // block is waited for before the last k-tile, below.)
                    const uint32_t* pass_flags =
                        p.ready + (p.tile_list[1 + tile].w >> 27) * (p.npr + p.npc);
                    wait_ready(pass_flags + bm / p.panel_rows, abort);
                    wait_ready(pass_flags + p.npr + bn / p.panel_cols, abort);
                    // the panels were written by the copy engine; order the TMA reads after
                    asm volatile("fence.proxy.async.global;\n" ::: "memory");
                }
                for (int kt = kt0; kt < kt1; ++kt, ++it) {
                    const int s = it % Cfg::STAGES;
                    const uint32_t r = static_cast<uint32_t>(it / Cfg::STAGES);
                    mbar_wait(&empty[s], (r & 1u) ^ 1u);
                    if constexpr (STREAMED) {
                        // The consumers read C in the epilogue, after this last stage's full
                        // barrier (release by this arrive, acquire by their wait): acquiring the
                        // C block's flag here orders those reads after its upload, and leaves
                        // the upload a whole tile of slack.
                        if (kt == ktiles - 1)
                            wait_ready(p.ready + p.tile_list[0].y * (p.npr + p.npc) +
                                           (bm / p.panel_rows) * p.npc + bn / p.panel_cols,
                                       abort);
                    }
                    mbar_arrive_expect_tx(&full[s], Cfg::STAGE_BYTES);
                    const uint32_t sa = smem_u32(ring + s * Cfg::STAGE_BYTES);
                    tma_load_2d(sa, &tmA, kt * Cfg::BK, bm, &full[s]);
#pragma unroll
                    for (int j = 0; j < Cfg::BN / 16; ++j)
                        tma_load_2d(sa + Cfg::A_BYTES + j * 2048, &tmB, bn + 16 * j, kt * Cfg::BK, &full[s]);
                }
            }
        }
        return;
    }

    // ---------------- consumers ----------------
    if constexpr (Cfg::REBALANCE)
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(CREGS));
    // SPLIT timeline trace (kw_dgemm_split_trace; p.tile_list is free in SPLIT mode): per virtual
    // CTA 40 u64 — start, SM id, (piece start, piece end) x 18, end — written by its first warp.
    // Compiled in only with -DKW_SPLIT_TRACE (the bookkeeping costs the two-group config spills).
#if defined(KW_SPLIT_TRACE)
    uint64_t* trace = nullptr;
    if constexpr (SPLIT) {
        if (p.tile_list && warp % Cfg::CONSUMERS == 0 && lane == 0)
            trace = reinterpret_cast<uint64_t*>(const_cast<int4*>(p.tile_list)) + static_cast<size_t>(ticket) * 40;
    }
    auto stamp = [&](int slot) {
        if (trace && slot < 40) {
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            trace[slot] = t;
        }
    };
    stamp(0);
    if (trace) {
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        trace[1] = smid;
    }
#else
    auto stamp = [](int) {};
#endif
    const int lw = warp - grp * Cfg::CONSUMERS; // warp within its consumer group
    const int wm = (lw / Cfg::WARPS_N) * Cfg::WM;
    const int wn = (lw % Cfg::WARPS_N) * Cfg::WN;
    const int g = lane >> 2, t = lane & 3;


    // Per-lane parts of the fragment addresses (bytes inside a stage).
    const uint32_t a_row = static_cast<uint32_t>(wm + g) * 128u;
    const uint32_t b_box = static_cast<uint32_t>(wn >> 4) * 2048u;
    uint32_t a_sw[4], b_even[4];
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
        const int k = 8 * (t >> 1) + 2 * ((t + ks) & 3) + (t & 1);
        a_sw[ks] = a_row + ((static_cast<uint32_t>((k >> 1) ^ g) << 4) | (static_cast<uint32_t>(k & 1) << 3));
        b_even[ks] = b_box + static_cast<uint32_t>(k) * 128u +
                     ((static_cast<uint32_t>((g >> 1) ^ (k & 7)) << 4) | ((g & 1) << 3));
    }
    auto load_frags = [&](const uint8_t* sa, int ks, double (&af)[Cfg::MT], double (&bf)[Cfg::NT]) {
        const uint8_t* sb = sa + Cfg::A_BYTES;
#pragma unroll
        for (int i = 0; i < Cfg::MT; ++i)
            af[i] = *reinterpret_cast<const double*>(sa + a_sw[ks] + i * 1024);
#pragma unroll
        for (int j = 0; j < Cfg::NT; ++j)
            bf[j] = *reinterpret_cast<const double*>(sb + (j >> 1) * 2048 + (b_even[ks] ^ ((j & 1) ? 64u : 0u)));
    };

    const bool c_vec = (p.ldc % 2 == 0) && (reinterpret_cast<uintptr_t>(p.c) % 16 == 0);
    int it0 = 0; // ring position of this tile's first k-tile
    for (int tile = first; tile < ntiles; tile += step) {
    int bm, bn, kt0, kt1;
    if (!origin(tile, bm, bn, kt0, kt1))
        continue;
    const int nkt = kt1 - kt0;
    // k-split (streamed only): this thread's accumulators of the tile, parked between passes;
    // item i of lane l at ((tile * CONSUMERS + warp) * MT*NT + i) * 32 + l (coalesced double2).
    double2* park = nullptr;
    if constexpr (STREAMED || KRANGE) {
        const size_t tid_tile = static_cast<size_t>(bm / Cfg::BM) * p.tiles_n + bn / Cfg::BN;
        park = reinterpret_cast<double2*>(p.partial) + (tid_tile * Cfg::CONSUMERS + lw) * (Cfg::MT * Cfg::NT) * 32 + lane;
        if (KRANGE && p.panel_cols > 0) // split-k: slice s parks into its own copy of the tile grid
            park += static_cast<size_t>(blockIdx.y) * p.tiles_m * p.tiles_n * Cfg::CONSUMERS * (Cfg::MT * Cfg::NT) * 32;
    }
    // split-k slices start from zero and always park (splitk_reduce sums them and runs the epilogue)
    const bool splitk = KRANGE && p.panel_cols > 0;
    // SPLIT: a tail piece reloads slot ticket - 1 (its head ran on the previous ticket), a head
    // piece parks into slot ticket.
    uint32_t* split_flags = SPLIT ? p.ready + 4 : nullptr;
    if constexpr (SPLIT) {
        const int slot = kt0 > 0 ? ticket - 1 : ticket;
        park = reinterpret_cast<double2*>(p.partial) +
               (static_cast<size_t>(slot) * Cfg::CONSUMERS + lw) * (Cfg::MT * Cfg::NT) * 32 + lane;
    }
    double acc[Cfg::MT][Cfg::NT][2];
#pragma unroll
    for (int i = 0; i < Cfg::MT; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::NT; ++j)
            acc[i][j][0] = acc[i][j][1] = 0.0;
    if constexpr (SPLIT) {
        if (kt0 > 0) {
            // wait for the head piece's park (flag of slot ticket - 1, this warp), bounded
            uint32_t* f = split_flags + (ticket - 1) * Cfg::CONSUMERS + lw;
            for (uint32_t spins = 0; ld_acquire_gpu(f) == 0; ++spins) {
                if (spins > (1u << 25)) { // ~30 s: never by construction (split_range)
                    split_abort(p.ready, lane);
                    break;
                }
                __nanosleep(256);
            }
#pragma unroll
            for (int i = 0; i < Cfg::MT; ++i)
#pragma unroll
                for (int j = 0; j < Cfg::NT; ++j) {
                    const double2 v = __ldcg(park + (i * Cfg::NT + j) * 32);
                    acc[i][j][0] = v.x;
                    acc[i][j][1] = v.y;
                }
            __syncwarp();
            if (lane == 0)
                *f = 0; // consumed: the flags are all zero again when the launch ends
        }
    }
    // One CTA per SM (SPLIT, MIN_BLOCKS 1) with a small warp tile: no co-resident CTA covers this
    // tile's epilogue, so its C reads are issued now into registers and land during the main loop
    // (C belongs to this tile alone). Larger warp tiles take the L2 prefetch below instead (split
    // 20 at 1280^3: 32.6 vs 31.8 TFLOP/s with the register copy).
    constexpr bool PREFETCH_C = KW_DGEMM_REG_PREFETCH_C && SPLIT && Cfg::MIN_BLOCKS == 1 && Cfg::MT * Cfg::NT <= 8;
    double2 cpre[PREFETCH_C ? Cfg::MT : 1][PREFETCH_C ? Cfg::NT : 1];
    if constexpr (PREFETCH_C) {
        if (kt1 == ktiles) {
#pragma unroll
            for (int i = 0; i < Cfg::MT; ++i) {
                const int row = bm + wm + i * 8 + g;
                const double* crow = p.c + (row < p.m ? row : 0) * p.ldc;
#pragma unroll
                for (int j = 0; j < Cfg::NT; ++j) {
                    const int col = bn + wn + j * 8 + 2 * t;
                    if (row < p.m && c_vec && col + 1 < p.n)
                        cpre[i][j] = __ldcs(reinterpret_cast<const double2*>(crow + col));
                    else {
                        cpre[i][j].x = (row < p.m && col < p.n) ? crow[col] : 0.0;
                        cpre[i][j].y = (row < p.m && col + 1 < p.n) ? crow[col + 1] : 0.0;
                    }
                }
            }
        }
    }
    // Other resident configurations: pull this tile's C block into L2 now (prefetch.global.L2,
    // no registers), so the epilogue's reads return from L2 rather than HBM.
    if constexpr (!PREFETCH_C && !STREAMED && KW_DGEMM_C_L2PF) {
        if (kt1 == ktiles && !splitk) {
            constexpr int SEGS = Cfg::WN / 16; // 128-byte lines per warp-tile row
            for (int idx = lane; idx < Cfg::WM * SEGS; idx += 32) {
                const int row = bm + wm + idx / SEGS, col = bn + wn + (idx % SEGS) * 16;
                if (row < p.m && col < p.n)
                    asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p.c + static_cast<size_t>(row) * p.ldc + col));
            }
        }
    }
    stamp(2 + 2 * tile);
    if constexpr (STREAMED || KRANGE) {
        if (kt0 > 0 && !splitk) {
#pragma unroll
            for (int i = 0; i < Cfg::MT; ++i)
#pragma unroll
                for (int j = 0; j < Cfg::NT; ++j) {
                    const double2 v = __ldcg(park + (i * Cfg::NT + j) * 32);
                    acc[i][j][0] = v.x;
                    acc[i][j][1] = v.y;
                }
        }
    }

    if constexpr (Cfg::PAIRED) {
        // A pair fragments: one double2 per (i, q) = k-steps 2q and 2q+1; B per k-step.
        const int a_bit = t >> 1, b_bit = t & 1;
        uint32_t a_sw2[2], b_ev[4];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int k_half = 4 * a_bit + 2 * b_bit + (a_bit ^ q); // k >> 1 for both k-steps of the pair
            a_sw2[q] = a_row + (static_cast<uint32_t>(k_half ^ g) << 4);
        }
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
            const int k = 8 * a_bit + 4 * b_bit + 2 * (a_bit ^ (ks >> 1)) + (ks & 1);
            b_ev[ks] = b_box + static_cast<uint32_t>(k) * 128u +
                       ((static_cast<uint32_t>((g >> 1) ^ (k & 7)) << 4) | ((g & 1) << 3));
        }
        auto load_a2 = [&](const uint8_t* sa, int q, double2 (&a2)[Cfg::MT]) {
#pragma unroll
            for (int i = 0; i < Cfg::MT; ++i)
                a2[i] = *reinterpret_cast<const double2*>(sa + a_sw2[q] + i * 1024);
        };
        auto load_b = [&](const uint8_t* sa, int ks, double (&bf)[Cfg::NT]) {
            const uint8_t* sb = sa + Cfg::A_BYTES;
#pragma unroll
            for (int j = 0; j < Cfg::NT; ++j)
                bf[j] = *reinterpret_cast<const double*>(sb + (j >> 1) * 2048 + (b_ev[ks] ^ ((j & 1) ? 64u : 0u)));
        };
        // A pairs double-buffered (one LDS.128 per row block covers two k-steps); B fragments
        // one k-step ahead — or, for small warp tiles (AHEAD2), two k-steps ahead from four
        // buffers and the next stage's first A pairs one k-step earlier: 8 DMMAs per k-step
        // are too few to cover a fragment load issued one step ahead.
        constexpr bool AHEAD2 = KW_DGEMM_AHEAD2 && Cfg::MT * Cfg::NT <= 8;
        if constexpr (AHEAD2) {
        double2 a2[2][Cfg::MT];
        double bf[4][Cfg::NT];
        if (nkt > 0) {
            const int s0 = it0 % Cfg::STAGES;
            mbar_wait(&full[s0], static_cast<uint32_t>(it0 / Cfg::STAGES) & 1u);
            load_a2(ring + s0 * Cfg::STAGE_BYTES, 0, a2[0]);
            load_b(ring + s0 * Cfg::STAGE_BYTES, 0, bf[0]);
            load_b(ring + s0 * Cfg::STAGE_BYTES, 1, bf[1]);
        }
        for (int kt = 0; kt < nkt; ++kt) {
            const int s = (it0 + kt) % Cfg::STAGES;
            const uint8_t* sa = ring + s * Cfg::STAGE_BYTES;
            const uint8_t* sa2 = sa;
            const bool more = kt + 1 < nkt;
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                const int q = ks >> 1, h = ks & 1;
                if (ks == 0)
                    load_a2(sa, 1, a2[1]);
                if (ks < 2)
                    load_b(sa, ks + 2, bf[ks + 2]);
                else if (more) {
                    if (ks == 2) {
                        const int s2 = (it0 + kt + 1) % Cfg::STAGES;
                        mbar_wait(&full[s2], static_cast<uint32_t>((it0 + kt + 1) / Cfg::STAGES) & 1u);
                        sa2 = ring + s2 * Cfg::STAGE_BYTES;
                        load_a2(sa2, 0, a2[0]); // a2[0] is idle during k-steps 2 and 3
                    }
                    load_b(sa2, ks - 2, bf[ks - 2]);
                }
#pragma unroll
                for (int i = 0; i < Cfg::MT; ++i)
#pragma unroll
                    for (int j = 0; j < Cfg::NT; ++j)
                        dmma_8x8x4(acc[i][j][0], acc[i][j][1], h ? a2[q][i].y : a2[q][i].x, bf[ks][j]);
                if (ks == 3) {
                    __syncwarp(); // stage s fully consumed (below)
                    if (lane == 0)
                        mbar_arrive(&empty[s]);
                }
            }
        }
        }
        else {
        double2 a2[2][Cfg::MT];
        double bf[2][Cfg::NT];
        if (nkt > 0) {
            const int s0 = it0 % Cfg::STAGES;
            mbar_wait(&full[s0], static_cast<uint32_t>(it0 / Cfg::STAGES) & 1u);
            load_a2(ring + s0 * Cfg::STAGE_BYTES, 0, a2[0]);
            load_b(ring + s0 * Cfg::STAGE_BYTES, 0, bf[0]);
        }
        for (int kt = 0; kt < nkt; ++kt) {
            const int s = (it0 + kt) % Cfg::STAGES;
            const uint8_t* sa = ring + s * Cfg::STAGE_BYTES;
            const uint8_t* sa2 = sa;
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                const int q = ks >> 1, h = ks & 1;
                const int bc = ks & 1, bn2 = bc ^ 1;
                if (ks == 0)
                    load_a2(sa, 1, a2[1]);
                if (ks < 3) {
                    load_b(sa, ks + 1, bf[bn2]);
                }
                else {
                    if (kt + 1 < nkt) {
                        const int s2 = (it0 + kt + 1) % Cfg::STAGES;
                        mbar_wait(&full[s2], static_cast<uint32_t>((it0 + kt + 1) / Cfg::STAGES) & 1u);
                        sa2 = ring + s2 * Cfg::STAGE_BYTES;
                        load_b(sa2, 0, bf[bn2]);
                        load_a2(sa2, 0, a2[0]); // a2[0] is idle during k-steps 2 and 3
                    }
                }
#pragma unroll
                for (int i = 0; i < Cfg::MT; ++i)
#pragma unroll
                    for (int j = 0; j < Cfg::NT; ++j)
                        dmma_8x8x4(acc[i][j][0], acc[i][j][1], h ? a2[q][i].y : a2[q][i].x, bf[bc][j]);
                if (ks == 3) {
                    // Release stage s only now: these DMMAs consumed its last fragments, so
                    // every LDS from it has returned. (An arrive right after issuing the LDS
                    // let the refill's TMA overwrite the stage under a still-pending LDS —
                    // seen as k-step-sized errors when tiles turn over quickly.)
                    __syncwarp();
                    if (lane == 0)
                        mbar_arrive(&empty[s]);
                }
            }
        }
        }
    }
    else {
    // Register double buffering: the fragments of the next k-step (or of the next stage's
    // first k-step) are loaded before the DMMAs of the current one are issued, so LDS latency
    // hides behind 32 DMMAs instead of stalling the warp.
    double af[2][Cfg::MT], bf[2][Cfg::NT];
    if (nkt > 0) {
        const int s0 = it0 % Cfg::STAGES;
        mbar_wait(&full[s0], static_cast<uint32_t>(it0 / Cfg::STAGES) & 1u);
        load_frags(ring + s0 * Cfg::STAGE_BYTES, 0, af[0], bf[0]);
    }
    for (int kt = 0; kt < nkt; ++kt) {
        const int s = (it0 + kt) % Cfg::STAGES;
        const uint8_t* sa = ring + s * Cfg::STAGE_BYTES;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
            const int cur = ks & 1, nxt = cur ^ 1;
            if (ks < 3) {
                load_frags(sa, ks + 1, af[nxt], bf[nxt]);
            }
            else {
                // wait for the next stage (if any) and prefetch its first k-step
                if (kt + 1 < nkt) {
                    const int s2 = (it0 + kt + 1) % Cfg::STAGES;
                    mbar_wait(&full[s2], static_cast<uint32_t>((it0 + kt + 1) / Cfg::STAGES) & 1u);
                    load_frags(ring + s2 * Cfg::STAGE_BYTES, 0, af[nxt], bf[nxt]);
                }
            }
#pragma unroll
            for (int i = 0; i < Cfg::MT; ++i)
#pragma unroll
                for (int j = 0; j < Cfg::NT; ++j)
                    dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[cur][i], bf[cur][j]);
            if (ks == 3) {
                // stage s fully consumed (see the paired loop): release it
                __syncwarp();
                if (lane == 0)
                    mbar_arrive(&empty[s]);
            }
        }
    }

    }
    it0 += nkt;
    if constexpr (SPLIT) {
        if (kt1 < ktiles) {
            // head piece: park the accumulators in slot `ticket`, then raise this warp's flag
#pragma unroll
            for (int i = 0; i < Cfg::MT; ++i)
#pragma unroll
                for (int j = 0; j < Cfg::NT; ++j)
                    __stcg(park + (i * Cfg::NT + j) * 32, make_double2(acc[i][j][0], acc[i][j][1]));
            __threadfence();
            __syncwarp();
            if (lane == 0)
                asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(split_flags + ticket * Cfg::CONSUMERS + lw),
                             "r"(1u)
                             : "memory");
            stamp(3 + 2 * tile);
            continue;
        }
    }
    if constexpr (STREAMED || KRANGE) {
        if (kt1 < ktiles || splitk) {
            // first pass of a k-split: park the accumulators; the second pass (streamed: same
            // CTA, same thread, later in this loop; k-range: the next launch) reloads them and
            // runs the epilogue
#pragma unroll
            for (int i = 0; i < Cfg::MT; ++i)
#pragma unroll
                for (int j = 0; j < Cfg::NT; ++j)
                    __stcg(park + (i * Cfg::NT + j) * 32, make_double2(acc[i][j][0], acc[i][j][1]));
            continue;
        }
    }

    // Epilogue, one 8-row block of the warp tile at a time: the block's C values are read before
    // any of them is written — interleaving load / compute / store serialises on the stores'
    // possible aliasing with the later loads (one L2 round trip per element pair, ~6 us per
    // 64 x 128 tile with the split timeline). A whole-tile batch would not fit the registers next
    // to the accumulators. (PREFETCH_C configurations read C at tile start instead.)
    constexpr int EB = Cfg::NT; // batch = the whole 8-row block (narrower batches measured no better)
#pragma unroll
    for (int i = 0; i < Cfg::MT; ++i) {
        const int row = bm + wm + i * 8 + g;
        if (row >= p.m)
            continue;
        double* crow = p.c + row * p.ldc;
#pragma unroll
        for (int j0 = 0; j0 < Cfg::NT; j0 += EB) {
        double2 old[EB];
#pragma unroll
        for (int jj = 0; jj < EB; ++jj) {
            const int j = j0 + jj;
            const int col = bn + wn + j * 8 + 2 * t;
            if constexpr (PREFETCH_C)
                old[jj] = cpre[i][j];
            else if (c_vec && col + 1 < p.n)
                old[jj] = *reinterpret_cast<const double2*>(crow + col);
            else {
                old[jj].x = col < p.n ? crow[col] : 0.0;
                old[jj].y = col + 1 < p.n ? crow[col + 1] : 0.0;
            }
        }
#pragma unroll
        for (int jj = 0; jj < EB; ++jj) {
            const int j = j0 + jj;
            const int col = bn + wn + j * 8 + 2 * t;
            const double x = __dadd_rn(__dmul_rn(p.alpha, acc[i][j][0]), __dmul_rn(p.beta, old[jj].x));
            const double y = __dadd_rn(__dmul_rn(p.alpha, acc[i][j][1]), __dmul_rn(p.beta, old[jj].y));
            if (c_vec && col + 1 < p.n)
                *reinterpret_cast<double2*>(crow + col) = make_double2(x, y);
            else {
                if (col < p.n)
                    crow[col] = x;
                if (col + 1 < p.n)
                    crow[col + 1] = y;
            }
        }
        }
    }
    if constexpr (STREAMED) {
        // this warp's share of the block is stored: make it visible to the copy engine, count it
        __syncwarp();
        if (lane == 0) {
            __threadfence_system();
            uint32_t* done = p.ready + p.tile_list[0].y * (p.npr + p.npc) + p.npr * p.npc;
            atomicAdd(done + (bm / p.panel_rows) * p.npc + bn / p.panel_cols, 1u);
        }
    }
    stamp(3 + 2 * tile);
    } // tile loop
    stamp(39);
}

using PFN_encodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled encode_fn()
{
    static PFN_encodeTiled fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled>(f);
        cudaGetLastError();
    });
    return fn;
}

// 2-D row-major fp64 matrix (rows x cols, ld elements) as a TMA map with box (16 cols, box_rows).
bool make_map(CUtensorMap* map, const double* base, size_t rows, size_t cols, size_t ld, uint32_t box_rows)
{
    PFN_encodeTiled enc = encode_fn();
    if (!enc)
        return false;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * sizeof(double))};
    const cuuint32_t box[2] = {16, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}


// 2-D row-major fp64 matrix as a TMA map with an unswizzled (box_cols x box_rows) box: the box
// lands dense in shared memory, row after row.
bool make_map_dense(CUtensorMap* map, const double* base, size_t rows, size_t cols, size_t ld, uint32_t box_cols,
                    uint32_t box_rows)
{
    PFN_encodeTiled enc = encode_fn();
    if (!enc)
        return false;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * sizeof(double))};
    const cuuint32_t box[2] = {box_cols, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// KW_DGEMM_PDL=0 launches the TMA kernels without programmatic dependent launch (A/B switch).
bool dgemm_pdl()
{
    static const bool on = [] {
        const char* e = std::getenv("KW_DGEMM_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

// PDL only where the early-launched grid cannot take free co-resident slots: a dependent CTA
// placed beside a short grid's CTAs fixes its SM before the grid drains and unbalances the next
// launch (measured: the 64 x 64 three-CTA tile at 1024^3 fell from 26.9 to 18.0 TFLOP/s).
template <class Cfg, bool STREAMED, bool SPLIT, bool KRANGE = false>
cudaError_t launch_tma_kernel(unsigned grid, cudaStream_t s, const CUtensorMap& ma, const CUtensorMap& mb,
                              const GemmParams& p, bool pdl, unsigned grid_y = 1)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid, grid_y);
    cfg.blockDim = dim3(Cfg::THREADS);
    cfg.dynamicSmemBytes = Cfg::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = (pdl && dgemm_pdl()) ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, dgemm_tma_kernel<Cfg, STREAMED, SPLIT, KRANGE>, ma, mb, p);
}

template <class Cfg, bool PERSISTENT = false, bool STREAMED = false>
kw_status launch_tma(cudaStream_t s, const GemmParams& p0);

// Tile configurations (the DGEMM half of the work-division sweep, BASELINE.json configs[4]).
using Cfg128 = TileCfg<128, 128, 16, 64, 32, 4>;          // 0: 8 warps of 64x32
using Cfg128k32 = TileCfg<128, 128, 32, 64, 32, 3>;       // 1
using Cfg128w16 = TileCfg<128, 128, 16, 32, 32, 4>;       // 2: 16 warps of 32x32
using Cfg128w16k32 = TileCfg<128, 128, 32, 32, 32, 3>;    // 3
using Cfg64 = TileCfg<64, 64, 16, 32, 32, 4, 2>;          // 4: 4 warps, several CTAs per SM
using Cfg128x64 = TileCfg<128, 64, 32, 32, 32, 4, 2>;     // 5: 8 warps of 32x32, 2 CTAs per SM
using Cfg64x128 = TileCfg<64, 128, 32, 32, 32, 4, 2>;     // 6

template <class Cfg>
kw_status launch_dmma(cudaStream_t s, const GemmParams& p0)
{
    GemmParams p = p0;
    p.tiles_m = static_cast<int>(kw::ceil_div(p.m, Cfg::BM));
    p.tiles_n = static_cast<int>(kw::ceil_div(p.n, Cfg::BN));
    const long long tiles = static_cast<long long>(p.tiles_m) * p.tiles_n;
    if (tiles > INT_MAX)
        return kw::usage("dgemm: problem too large for the tile grid");
    const bool vec16 = (p.lda % 2 == 0) && (p.ldb % 2 == 0) && (reinterpret_cast<uintptr_t>(p.a) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(p.b) % 16 == 0);
    auto kern = vec16 ? dgemm_dmma_kernel<Cfg, true> : dgemm_dmma_kernel<Cfg, false>;
    const kw_status st = ensure_smem(reinterpret_cast<const void*>(kern), Cfg::SMEM, "dgemm: cudaFuncSetAttribute");
    if (st != KW_OK)
        return st;
    kern<<<static_cast<unsigned>(tiles), Cfg::THREADS, Cfg::SMEM, s>>>(p);
    kw::g_launches.fetch_add(1, std::memory_order_relaxed);
    return KW_OK;
}

// ------------------------------------------------------------------------------------------
// K3: GemmNaiveKernel on the GPU — bit-exact. The division covers the outputs of gemm.cpp:13-22
// (grid thread (r, c) owns rows [r*er, r*er+er) x cols [c*ec, c*ec+ec), clamped at (m, n)); per
// element one ascending-p dot product from +0.0 with separately rounded products and sums, then
// the two-rounding epilogue (gemm.cpp:30-36). Axis rule: the last (fastest) work-division
// component is CUDA x.
// ------------------------------------------------------------------------------------------
__global__ void dgemm_naive_kernel(GemmParams p, int er, int ec)
{
    // Block (by, bx) covers exactly the reference blocks' outputs: rows [by*TY*er, +TY*er) x
    // cols [bx*TX*ec, +TX*ec) (gemm.cpp:13-22 summed over the block's threads). Inside the block
    // the elements go to lanes in column order, so consecutive lanes read consecutive B columns
    // and write consecutive C columns (coalesced) whatever the division — the reference's
    // gemmNaiveWorkDiv puts its threads along rows. No bit depends on which thread computes an
    // element: each one is its own ascending-p dot product.
    const long long tile_rows = static_cast<long long>(blockDim.y) * er;
    const long long tile_cols = static_cast<long long>(blockDim.x) * ec;
    const long long row0 = static_cast<long long>(blockIdx.y) * tile_rows;
    const long long col0 = static_cast<long long>(blockIdx.x) * tile_cols;
    if (row0 >= p.m || col0 >= p.n)
        return;
    const long long rows = p.m - row0 < tile_rows ? p.m - row0 : tile_rows;
    const long long cols = p.n - col0 < tile_cols ? p.n - col0 : tile_cols;
    const long long nthr = static_cast<long long>(blockDim.x) * blockDim.y;
    const long long tid = static_cast<long long>(threadIdx.y) * blockDim.x + threadIdx.x;
    for (long long e = tid; e < rows * cols; e += nthr) {
        const long long row = row0 + e / cols, col = col0 + e % cols;
        double acc = 0.0;
        const double* ap = p.a + row * p.lda;
        const double* bp = p.b + col;
        for (int q = 0; q < p.k; ++q)
            acc = __dadd_rn(acc, __dmul_rn(ap[q], bp[q * p.ldb]));
        double* cp = p.c + row * p.ldc + col;
        *cp = __dadd_rn(__dmul_rn(p.alpha, acc), __dmul_rn(p.beta, *cp));
    }
}


// ------------------------------------------------------------------------------------------
// K2-bitwise: tiled DGEMM that is BITWISE equal to gemmReference (reference.cpp:14-26) and to
// the reference's own GemmTiledKernel (gemm.cpp:40-118, which test_kernels.cpp:208-230 pins
// bitwise to the naive kernel). Every output element is accumulated from +0.0 over k = 0..K-1
// in ascending order with separately rounded products and sums (DMUL then DADD, never DFMA),
// then fl(fl(alpha*acc) + fl(beta*c)). Padded k never enters a sum. FP64 pipe bound: two
// pipe operations per term, so at most half the DFMA rate.
//   block tile 128 x 128, k-tile 32 (2 stages), 256 threads; thread (ty, tx) owns C[ty + 16i][tx + 16j],
//   i, j < 8 (64 independent accumulation chains); A staged row-major with a (BK + 2)-double row
//   pitch (two rows read by one warp land in different banks), B row-major; STAGES-deep cp.async ring.
// ------------------------------------------------------------------------------------------
// Thread (ty, tx) of 16 x 16 owns C[ty + 16i][tx + 16j], i < 8, j < NJ; block tile 128 x 16*NJ.
template <int NJ_, int MIN_BLOCKS_, int BK_ = 16, int STAGES_ = 3>
struct BwCfg {
    static constexpr int NJ = NJ_, MIN_BLOCKS = MIN_BLOCKS_;
    static constexpr int BM = 128, BN = 16 * NJ, BK = BK_, THREADS = 256, STAGES = STAGES_;
    static constexpr int A_LD = BK + 2; // doubles: two rows a warp reads land in different banks
    static constexpr int A_STAGE = BM * A_LD, B_STAGE = BK * BN;
    static constexpr size_t SMEM = static_cast<size_t>(STAGES) * (A_STAGE + B_STAGE) * sizeof(double);
};
// 64 chains per thread, one CTA per SM, k-tile 32 in a 2-stage ring: half the block barriers of
// k-tile 16 (+1.2 %, tools/bitwise_ab.py: 16.35 vs 16.16 TFLOP/s at 8192^3; a 4th stage gains
// nothing). A 128 x 64 tile at two CTAs per SM measured 1.3 % slower: FP64-pipe bound.
using Bw128 = BwCfg<8, 1, 32, 2>;

template <class Cfg, bool VEC16>
__device__ __forceinline__ void bw_load_stage(const GemmParams& p, double* sA, double* sB, int bm, int bn, int k0,
                                              int tid)
{
#pragma unroll
    for (int it = 0; it < (Cfg::BM * Cfg::BK / 2) / Cfg::THREADS; ++it) {
        const int c = tid + it * Cfg::THREADS;
        const int row = c / (Cfg::BK / 2), kc = c % (Cfg::BK / 2);
        const int gm = bm + row, gk = k0 + kc * 2;
        int valid = 0;
        if (gm < p.m) {
            valid = p.k - gk;
            valid = valid < 0 ? 0 : (valid > 2 ? 2 : valid);
        }
        const double* src = valid > 0 ? p.a + gm * p.lda + gk : p.a;
        const uint32_t dst = smem_u32(sA + row * Cfg::A_LD + kc * 2);
        if (VEC16) {
            cp_async16(dst, src, valid * 8);
        }
        else {
            cp_async8(dst, src, valid >= 1 ? 8 : 0);
            cp_async8(dst + 8, valid >= 2 ? src + 1 : p.a, valid >= 2 ? 8 : 0);
        }
    }
#pragma unroll
    for (int it = 0; it < (Cfg::BK * Cfg::BN / 2) / Cfg::THREADS; ++it) {
        const int c = tid + it * Cfg::THREADS;
        const int row = c / (Cfg::BN / 2), nc = c % (Cfg::BN / 2);
        const int gk = k0 + row, gn = bn + nc * 2;
        int valid = 0;
        if (gk < p.k) {
            valid = p.n - gn;
            valid = valid < 0 ? 0 : (valid > 2 ? 2 : valid);
        }
        const double* src = valid > 0 ? p.b + gk * p.ldb + gn : p.b;
        const uint32_t dst = smem_u32(sB + row * Cfg::BN + nc * 2);
        if (VEC16) {
            cp_async16(dst, src, valid * 8);
        }
        else {
            cp_async8(dst, src, valid >= 1 ? 8 : 0);
            cp_async8(dst + 8, valid >= 2 ? src + 1 : p.b, valid >= 2 ? 8 : 0);
        }
    }
}

template <class Cfg>
__device__ __forceinline__ void bw_kstep(double (&acc)[8][Cfg::NJ], const double* a_s, const double* b_s, int kk)
{
    double a[8], b[Cfg::NJ];
#pragma unroll
    for (int i = 0; i < 8; ++i)
        a[i] = a_s[i * 16 * Cfg::A_LD + kk];
#pragma unroll
    for (int j = 0; j < Cfg::NJ; ++j)
        b[j] = b_s[kk * Cfg::BN + j * 16];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::NJ; ++j)
            acc[i][j] = __dadd_rn(acc[i][j], __dmul_rn(a[i], b[j])); // never contracted to DFMA
}

template <class Cfg, bool VEC16>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MIN_BLOCKS) dgemm_bitwise_kernel(GemmParams p)
{
    extern __shared__ __align__(128) double smem[];
    double* sA = smem;
    double* sB = smem + Cfg::STAGES * Cfg::A_STAGE;
    constexpr int GROUP = 8;
    const int tile = blockIdx.x;
    const int per_group = GROUP * p.tiles_n;
    const int group = tile / per_group;
    const int first_m = group * GROUP;
    const int gsize = (p.tiles_m - first_m) < GROUP ? (p.tiles_m - first_m) : GROUP;
    const int in_group = tile - group * per_group;
    const int bm = (first_m + in_group % gsize) * Cfg::BM;
    const int bn = (in_group / gsize) * Cfg::BN;
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;

    double acc[8][Cfg::NJ];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::NJ; ++j)
            acc[i][j] = 0.0;

    const int ktiles = (p.k + Cfg::BK - 1) / Cfg::BK;
#pragma unroll
    for (int s = 0; s < Cfg::STAGES - 1; ++s) {
        if (s < ktiles)
            bw_load_stage<Cfg, VEC16>(p, sA + s * Cfg::A_STAGE, sB + s * Cfg::B_STAGE, bm, bn, s * Cfg::BK, tid);
        cp_async_commit();
    }
    for (int kt = 0; kt < ktiles; ++kt) {
        cp_async_wait<Cfg::STAGES - 2>();
        __syncthreads();
        {
            const int nk = kt + Cfg::STAGES - 1;
            if (nk < ktiles) {
                const int s = nk % Cfg::STAGES;
                bw_load_stage<Cfg, VEC16>(p, sA + s * Cfg::A_STAGE, sB + s * Cfg::B_STAGE, bm, bn, nk * Cfg::BK, tid);
            }
            cp_async_commit();
        }
        const int s = kt % Cfg::STAGES;
        const double* a_s = sA + s * Cfg::A_STAGE + ty * Cfg::A_LD;
        const double* b_s = sB + s * Cfg::B_STAGE + tx;
        const int kend = (p.k - kt * Cfg::BK) < Cfg::BK ? (p.k - kt * Cfg::BK) : Cfg::BK; // no padded terms
        if (kend == Cfg::BK) {
#pragma unroll
            for (int kk = 0; kk < Cfg::BK; ++kk)
                bw_kstep<Cfg>(acc, a_s, b_s, kk);
        }
        else {
            for (int kk = 0; kk < kend; ++kk)
                bw_kstep<Cfg>(acc, a_s, b_s, kk);
        }
    }
    cp_async_wait<0>();
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int row = bm + ty + 16 * i;
        if (row >= p.m)
            continue;
        double* crow = p.c + row * p.ldc;
#pragma unroll
        for (int j = 0; j < Cfg::NJ; ++j) {
            const int col = bn + tx + 16 * j;
            if (col < p.n)
                crow[col] = __dadd_rn(__dmul_rn(p.alpha, acc[i][j]), __dmul_rn(p.beta, crow[col]));
        }
    }
}

// Bit-exact mode, warp-specialised: the same per-element arithmetic as dgemm_bitwise_kernel
// (acc = dadd(acc, dmul(a, b)) over k ascending from +0.0, padded k never summed, two-rounding
// epilogue), but the k-tiles arrive by TMA in an mbarrier ring filled by one producer lane, so the
// 8 consumer warps never meet at a block barrier: a warp waiting for a stage leaves the FP64 pipe
// to the other warp of its sub-partition. Consumer warp w owns rows w + 8i (i < 16) and lane l
// columns l + 32j (j < 4): the A operand of a k-step is one broadcast address per warp (no bank
// conflicts on a dense TMA box), B is 32 consecutive doubles.
struct BwTmaCfg {
    static constexpr int BM = 128, BN = 128, BK = 32, STAGES = 3, CONSUMERS = 8;
    static constexpr int MI = 16, NJ = 4; // per-thread outputs: MI rows x NJ columns
    static constexpr int THREADS = 32 * (CONSUMERS + 4);
    static constexpr int PRODUCER_REGS = 40, CONSUMER_REGS = 232; // 4*40 + 8*232 <= 12 * 168
    static constexpr uint32_t A_BYTES = BM * BK * 8, B_BYTES = BK * BN * 8, STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr size_t SMEM = 1024 + static_cast<size_t>(STAGES) * STAGE_BYTES + 2 * STAGES * sizeof(uint64_t);
    static_assert(4 * PRODUCER_REGS + CONSUMERS * CONSUMER_REGS <= 12 * 168, "register pool overcommitted");
};

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, 1)
    dgemm_bitwise_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                             GemmParams p)
{
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
    uint64_t* empty = full + Cfg::STAGES;
    constexpr int GROUP = 8;
    const int tile = blockIdx.x;
    const int per_group = GROUP * p.tiles_n;
    const int group = tile / per_group;
    const int first_m = group * GROUP;
    const int gsize = (p.tiles_m - first_m) < GROUP ? (p.tiles_m - first_m) : GROUP;
    const int in_group = tile - group * per_group;
    const int bm = (first_m + in_group % gsize) * Cfg::BM;
    const int bn = (in_group / gsize) * Cfg::BN;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < Cfg::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], Cfg::CONSUMERS);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int ktiles = (p.k + Cfg::BK - 1) / Cfg::BK;

    if (warp >= Cfg::CONSUMERS) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(Cfg::PRODUCER_REGS));
        if (warp == Cfg::CONSUMERS && lane == 0) {
            tma_prefetch_desc(&tmA);
            tma_prefetch_desc(&tmB);
            for (int kt = 0; kt < ktiles; ++kt) {
                const int s = kt % Cfg::STAGES;
                mbar_wait(&empty[s], (static_cast<uint32_t>(kt / Cfg::STAGES) & 1u) ^ 1u);
                mbar_arrive_expect_tx(&full[s], Cfg::STAGE_BYTES);
                const uint32_t sa = smem_u32(smem + s * Cfg::STAGE_BYTES);
                tma_load_2d(sa, &tmA, kt * Cfg::BK, bm, &full[s]);
                tma_load_2d(sa + Cfg::A_BYTES, &tmB, bn, kt * Cfg::BK, &full[s]);
            }
        }
        return;
    }
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(Cfg::CONSUMER_REGS));

    double acc[Cfg::MI][Cfg::NJ];
#pragma unroll
    for (int i = 0; i < Cfg::MI; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::NJ; ++j)
            acc[i][j] = 0.0;
    for (int kt = 0; kt < ktiles; ++kt) {
        const int s = kt % Cfg::STAGES;
        mbar_wait(&full[s], static_cast<uint32_t>(kt / Cfg::STAGES) & 1u);
        const double* a_s = reinterpret_cast<const double*>(smem + s * Cfg::STAGE_BYTES) + warp * Cfg::BK;
        const double* b_s = reinterpret_cast<const double*>(smem + s * Cfg::STAGE_BYTES + Cfg::A_BYTES) + lane;
        const int kend = (p.k - kt * Cfg::BK) < Cfg::BK ? (p.k - kt * Cfg::BK) : Cfg::BK; // no padded terms
        auto kstep = [&](int kk) {
            double a[Cfg::MI], b[Cfg::NJ];
#pragma unroll
            for (int i = 0; i < Cfg::MI; ++i)
                a[i] = a_s[i * 8 * Cfg::BK + kk];
#pragma unroll
            for (int j = 0; j < Cfg::NJ; ++j)
                b[j] = b_s[kk * Cfg::BN + 32 * j];
#pragma unroll
            for (int i = 0; i < Cfg::MI; ++i)
#pragma unroll
                for (int j = 0; j < Cfg::NJ; ++j)
                    acc[i][j] = __dadd_rn(acc[i][j], __dmul_rn(a[i], b[j])); // never contracted to DFMA
        };
        if (kend == Cfg::BK) {
#pragma unroll 4
            for (int kk = 0; kk < Cfg::BK; ++kk)
                kstep(kk);
        }
        else {
            for (int kk = 0; kk < kend; ++kk)
                kstep(kk);
        }
        // every value read from stage s has been consumed by the arithmetic above
        __syncwarp();
        if (lane == 0)
            mbar_arrive(&empty[s]);
    }
#pragma unroll
    for (int i = 0; i < Cfg::MI; ++i) {
        const int row = bm + warp + 8 * i;
        if (row >= p.m)
            continue;
        double* crow = p.c + row * p.ldc;
        double old[Cfg::NJ]; // the row's C values read before any is written (see the DMMA kernel)
#pragma unroll
        for (int j = 0; j < Cfg::NJ; ++j) {
            const int col = bn + lane + 32 * j;
            old[j] = col < p.n ? crow[col] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < Cfg::NJ; ++j) {
            const int col = bn + lane + 32 * j;
            if (col < p.n)
                crow[col] = __dadd_rn(__dmul_rn(p.alpha, acc[i][j]), __dmul_rn(p.beta, old[j]));
        }
    }
}

template <class Cfg>
kw_status launch_bitwise_cfg(cudaStream_t s, const GemmParams& p0)
{
    GemmParams p = p0;
    p.tiles_m = static_cast<int>(kw::ceil_div(p.m, Cfg::BM));
    p.tiles_n = static_cast<int>(kw::ceil_div(p.n, Cfg::BN));
    const long long tiles = static_cast<long long>(p.tiles_m) * p.tiles_n;
    if (tiles > INT_MAX)
        return kw::usage("dgemm: problem too large for the tile grid");
    const bool vec16 = (p.lda % 2 == 0) && (p.ldb % 2 == 0) && (reinterpret_cast<uintptr_t>(p.a) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(p.b) % 16 == 0);
    auto kern = vec16 ? dgemm_bitwise_kernel<Cfg, true> : dgemm_bitwise_kernel<Cfg, false>;
    const kw_status st =
        ensure_smem(reinterpret_cast<const void*>(kern), Cfg::SMEM, "dgemm_bitwise: cudaFuncSetAttribute");
    if (st != KW_OK)
        return st;
    kern<<<static_cast<unsigned>(tiles), Cfg::THREADS, Cfg::SMEM, s>>>(p);
    kw::g_launches.fetch_add(1, std::memory_order_relaxed);
    return KW_OK;
}

kw_status launch_bitwise_tma(cudaStream_t s, const GemmParams& p0)
{
    using Cfg = BwTmaCfg;
    GemmParams p = p0;
    p.tiles_m = static_cast<int>(kw::ceil_div(p.m, Cfg::BM));
    p.tiles_n = static_cast<int>(kw::ceil_div(p.n, Cfg::BN));
    const long long tiles = static_cast<long long>(p.tiles_m) * p.tiles_n;
    if (tiles > INT_MAX)
        return kw::usage("dgemm: problem too large for the tile grid");
    CUtensorMap ma, mb;
    if (!make_map_dense(&ma, p.a, p.m, p.k, p.lda, Cfg::BK, Cfg::BM) ||
        !make_map_dense(&mb, p.b, p.k, p.n, p.ldb, Cfg::BN, Cfg::BK))
        return launch_bitwise_cfg<Bw128>(s, p0);
    const kw_status st = ensure_smem(reinterpret_cast<const void*>(dgemm_bitwise_tma_kernel<Cfg>), Cfg::SMEM,
                                     "dgemm_bitwise: cudaFuncSetAttribute");
    if (st != KW_OK)
        return st;
    dgemm_bitwise_tma_kernel<Cfg><<<static_cast<unsigned>(tiles), Cfg::THREADS, Cfg::SMEM, s>>>(ma, mb, p);
    kw::g_launches.fetch_add(1, std::memory_order_relaxed);
    return KW_OK;
}

kw_status launch_bitwise(cudaStream_t s, const GemmParams& p)
{
    const char* e = std::getenv("KW_BW_TMA");
    const bool tma = !(e && e[0] == '0') && p.k > 0 && (p.lda * 8) % 16 == 0 && (p.ldb * 8) % 16 == 0 &&
                     reinterpret_cast<uintptr_t>(p.a) % 16 == 0 && reinterpret_cast<uintptr_t>(p.b) % 16 == 0 &&
                     encode_fn() != nullptr;
    return tma ? launch_bitwise_tma(s, p) : launch_bitwise_cfg<Bw128>(s, p);
}

kw_status validate_gemm(size_t m, size_t n, size_t k, const double* A, size_t lda, const double* B, size_t ldb,
                        const double* C, size_t ldc)
{
    if (m > INT_MAX || n > INT_MAX || k > INT_MAX)
        return kw::usage("dgemm: extents exceed 2^31-1");
    if (m == 0 || n == 0)
        return KW_OK;
    if (!A && k > 0)
        return kw::usage("dgemm: null A");
    if (!B && k > 0)
        return kw::usage("dgemm: null B");
    if (!C)
        return kw::usage("dgemm: null C");
    if (k > 0 && lda < k)
        return kw::usage("dgemm: lda smaller than k");
    if (k > 0 && ldb < n)
        return kw::usage("dgemm: ldb smaller than n");
    if (ldc < n)
        return kw::usage("dgemm: ldc smaller than n");
    return KW_OK;
}

// Picks the DMMA tile configuration named by a GPU work division (gemmTiledWorkDiv for the
// GPU back-end): threadsPerBlock x elementsPerThread == (BM, BN) and one block per tile.
kw_status tile_from_wd(const kw_workdiv* wd, size_t m, size_t n, int* tile)
{
    if (wd == nullptr) {
        *tile = 128;
        return KW_OK;
    }
    if (wd->dim != 2)
        return kw::usage("dgemm: the tiled kernel runs on a 2-D (rows, cols) work division");
    const size_t tm = wd->threads[0] * wd->elems[0], tn = wd->threads[1] * wd->elems[1];
    const size_t thr = wd->threads[0] * wd->threads[1];
    int t = 0;
    if (tm == 128 && tn == 128 && thr == static_cast<size_t>(Cfg128::THREADS))
        t = 128;
    else if (tm == 64 && tn == 64 && thr == static_cast<size_t>(Cfg64::THREADS))
        t = 64;
    else
        return kw::usage("dgemm: unsupported GPU tile configuration (supported: 128x128 tile with 256 threads, "
                         "64x64 tile with 128 threads; use gemmTiledWorkDiv(GpuCudaRt, m, n, tile))");
    if (wd->blocks[0] * tm < m || wd->blocks[1] * tn < n)
        return kw::usage("dgemm: work division does not cover the m x n output");
    *tile = t;
    return KW_OK;
}

int sm_count() // of the current device (cached per device)
{
    static std::atomic<int> cache[64] = {};
    int d = 0;
    cudaGetDevice(&d);
    if (d < 0 || d >= 64)
        d = 0;
    int v = cache[d].load(std::memory_order_relaxed);
    if (v == 0) {
        v = 148;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d) != cudaSuccess) {
            cudaGetLastError();
            v = 148;
        }
        cache[d].store(v, std::memory_order_relaxed);
    }
    return v;
}

// Tile-rows per raster group of resident launches (KW_DGEMM_GROUP; default 16: 8192^3 reads
// 9.2 GB of DRAM instead of 11.6 with 8, same rate — profiles/dgemm_raster_group_r02.txt).
int dgemm_group()
{
    static const int g = [] {
        const char* e = std::getenv("KW_DGEMM_GROUP");
        const int v = e ? std::atoi(e) : 0;
        return v > 1 && v <= 1024 ? v : 16;
    }();
    return g;
}

template <class Cfg, bool PERSISTENT, bool STREAMED>
kw_status launch_tma(cudaStream_t s, const GemmParams& p0)
{
    GemmParams p = p0;
    if constexpr (!STREAMED)
        p.panel_rows = dgemm_group();
    p.tiles_m = static_cast<int>(kw::ceil_div(p.m, Cfg::BM));
    p.tiles_n = static_cast<int>(kw::ceil_div(p.n, Cfg::BN));
    const long long tiles = static_cast<long long>(p.tiles_m) * p.tiles_n;
    if (tiles > INT_MAX)
        return kw::usage("dgemm: problem too large for the tile grid");
    if (!tma_eligible(p)) {
        if (p.ready)
            return kw::usage("dgemm (streamed): operands not TMA-addressable");
        return launch_dmma<Cfg128>(s, p0); // unaligned operands: cp.async kernel
    }
    CUtensorMap ma, mb;
    if (!make_map(&ma, p.a, p.m, p.k, p.lda, Cfg::BM) || !make_map(&mb, p.b, p.k, p.n, p.ldb, 16)) {
        if (p.ready)
            return kw::usage("dgemm (streamed): tensor map encoding failed");
        return launch_dmma<Cfg128>(s, p0);
    }
    const kw_status st = ensure_smem(reinterpret_cast<const void*>(dgemm_tma_kernel<Cfg, STREAMED, false>), Cfg::SMEM,
                                     "dgemm: cudaFuncSetAttribute");
    if (st != KW_OK)
        return st;
    const long long resident = static_cast<long long>(sm_count()) * Cfg::MIN_BLOCKS;
    const long long ctas = (tiles + Cfg::GROUPS - 1) / Cfg::GROUPS; // a CTA serves GROUPS tiles at a time
    const unsigned grid = static_cast<unsigned>(PERSISTENT && ctas > resident ? resident : ctas);
    if constexpr (STREAMED) {
        dgemm_tma_kernel<Cfg, true, false><<<grid, Cfg::THREADS, Cfg::SMEM, s>>>(ma, mb, p);
    }
    else {
        if (cudaError_t e = launch_tma_kernel<Cfg, false, false>(grid, s, ma, mb, p, grid >= resident))
            return kw::cuda_fail("dgemm: launch", e);
    }
    kw::g_launches.fetch_add(1, std::memory_order_relaxed);
    return KW_OK;
}

using Tma128 = TmaCfg<128, 128, 64, 32, 6>;   // 7: 8 consumer warps + 1 producer
using Tma128s4 = TmaCfg<128, 128, 64, 32, 4>; // 8
using Tma64x128 = TmaCfg<64, 128, 32, 32, 6>; // 9: 8 consumers of 32x32
using Tma128x64 = TmaCfg<128, 64, 64, 32, 6>; // 10: 4 consumers
using Tma128s7 = TmaCfg<128, 128, 64, 32, 7>; // 11: 7-stage ring (224 KiB)
using Tma128x64x2 = TmaCfg<128, 64, 64, 32, 4, 2>; // 12: two CTAs per SM, 4 consumers each
using Tma64x128x2 = TmaCfg<64, 128, 64, 32, 4, 2>; // 13
using Tma128p = TmaCfg<128, 128, 64, 32, 6, 1, true>;       // 14: LDS.128 paired A fragments
using Tma64x128x2p = TmaCfg<64, 128, 64, 32, 4, 2, true>;   // 16: paired, two CTAs per SM
using Tma64x64x3p = TmaCfg<64, 64, 32, 32, 4, 3, true>;     // 17: paired, three CTAs per SM
using Split64w8 = TmaCfg<64, 64, 32, 16, 8, 1, true>;       // 18: SPLIT, 8 consumers of 32x16, 1 CTA/SM
using Split64w4 = TmaCfg<64, 64, 32, 32, 8, 1, true>;       // 19: SPLIT, 4 consumers of 32x32
using Split64x128w8 = TmaCfg<64, 128, 32, 32, 6, 1, true>;  // 20: SPLIT, 8 consumers of 32x32
using Split64w8t = TmaCfg<64, 64, 16, 32, 8, 1, true>;      // 23: SPLIT, 8 consumers of 16x32
// 25 / 26: two consumer groups of config 16's geometry (64 x 128 tiles, 4 warps of 64 x 32) in one
// CTA per SM, each with its own 4-stage ring and producer lane — SPLIT walk / data-parallel.
using Pair64x128 = TmaCfg<64, 128, 64, 32, 4, 1, true, 2>;
using Tma32p = TmaCfg<32, 32, 16, 16, 8, 3, true>;   // 28: 32 x 32 tiles, 4 warps of 16 x 16, 3 CTAs/SM
using Tma32x64p = TmaCfg<32, 64, 16, 32, 8, 2, true>; // 29: 32 x 64 tiles, 4 warps of 16 x 32, 2 CTAs/SM
// (16 consumer warps of 32x32 were measured out: 104 registers per consumer spill.)

// ---- SPLIT launches: per-stream scratch (ticket, abort pointer, flags, park slots) ----------
struct SplitScratch {
    int device = -1;
    cudaStream_t stream = nullptr;
    uint32_t* flags = nullptr; // [u64 ticket][u64 abort pointer][flags]
    size_t flag_words = 0;
    double* park = nullptr;
    size_t park_bytes = 0;
    uint32_t* abort_host = nullptr; // mapped pinned: [u32 abort][pad][u64 its device address]
    long long last_grid = 0;        // tickets are (counter % grid): the counter must be a multiple
                                    // of the grid at every launch (start order = ticket order)
};
std::mutex g_split_mu;
std::vector<SplitScratch*> g_split;

kw_status split_scratch(cudaStream_t s, long long grid, size_t flag_words, size_t park_bytes, uint32_t** flags,
                        double** park)
{
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(g_split_mu);
    SplitScratch* sc = nullptr;
    for (SplitScratch* x : g_split)
        if (x->device == dev && x->stream == s)
            sc = x;
    if (!sc) {
        sc = new SplitScratch;
        sc->device = dev;
        sc->stream = s;
        g_split.push_back(sc);
    }
    cudaError_t e = cudaSuccess;
    if (!sc->abort_host) {
        void* h = nullptr;
        e = cudaHostAlloc(&h, 16, cudaHostAllocMapped | cudaHostAllocPortable);
        if (e != cudaSuccess)
            return kw::cuda_fail("dgemm split: pinned abort word", e);
        sc->abort_host = static_cast<uint32_t*>(h);
        void* d = nullptr;
        cudaHostGetDevicePointer(&d, h, 0);
        sc->abort_host[0] = 0;
        *reinterpret_cast<void**>(sc->abort_host + 2) = d;
    }
    if (sc->flag_words < flag_words || sc->park_bytes < park_bytes) {
        cudaStreamSynchronize(s); // the previous launches on this stream still use the old scratch
        if (sc->flag_words < flag_words) {
            cudaFree(sc->flags);
            sc->flags = nullptr;
            sc->flag_words = 0;
            e = cudaMalloc(&sc->flags, flag_words * sizeof(uint32_t));
            if (e == cudaSuccess)
                e = cudaMemsetAsync(sc->flags, 0, flag_words * sizeof(uint32_t), s);
            if (e == cudaSuccess) // the kernel finds the abort word through the scratch
                e = cudaMemcpyAsync(sc->flags + 2, sc->abort_host + 2, 8, cudaMemcpyHostToDevice, s);
            if (e != cudaSuccess)
                return kw::cuda_fail("dgemm split: flag scratch", e);
            sc->flag_words = flag_words;
        }
        if (sc->park_bytes < park_bytes) {
            cudaFree(sc->park);
            sc->park = nullptr;
            sc->park_bytes = 0;
            e = cudaMalloc(&sc->park, park_bytes);
            if (e != cudaSuccess)
                return kw::cuda_fail("dgemm split: park scratch", e);
            sc->park_bytes = park_bytes;
        }
    }
    if (sc->last_grid != grid) {
        // A launch with another grid size left the ticket counter at a multiple of ITS grid:
        // restart it, stream-ordered after the previous launch, so tickets again follow start
        // order (a rotated order would let a started CTA wait on one that has not started).
        e = cudaMemsetAsync(sc->flags, 0, 8, s);
        if (e != cudaSuccess)
            return kw::cuda_fail("dgemm split: ticket reset", e);
        sc->last_grid = grid;
    }
    *flags = sc->flags;
    *park = sc->park;
    return KW_OK;
}

// Debug/measurement: a device buffer the next SPLIT launches stamp their timeline into
// (kw_dgemm_split_trace; 40 u64 per virtual CTA), or nullptr. Only a library built with
// -DKW_SPLIT_TRACE (KW_EXTRA_NVCC_FLAGS) stamps.
std::atomic<void*> g_split_trace{nullptr};

// One persistent CTA per SM over equal (tile, k-tile) ranges (dgemm_tma_kernel SPLIT).
template <class Cfg>
kw_status launch_split(cudaStream_t s, const GemmParams& p0)
{
    static_assert(Cfg::PAIRED, "split: paired k-map configurations only");
    GemmParams p = p0;
    p.tiles_m = static_cast<int>(kw::ceil_div(p.m, Cfg::BM));
    p.tiles_n = static_cast<int>(kw::ceil_div(p.n, Cfg::BN));
    const long long tiles = static_cast<long long>(p.tiles_m) * p.tiles_n;
    const long long G = static_cast<long long>(sm_count()) * Cfg::MIN_BLOCKS; // every CTA resident
    const long long VG = G * Cfg::GROUPS;                                      // virtual CTAs
    const long long ktiles = kw::ceil_div(p.k, Cfg::BK);
    // every range must span at least one whole tile (a tile is then split at most once)
    if (tiles < VG || ktiles < 2 || tiles * ktiles > INT_MAX || !tma_eligible(p))
        return launch_tma<Tma64x64x3p>(s, p0);
    CUtensorMap ma, mb;
    if (!make_map(&ma, p.a, p.m, p.k, p.lda, Cfg::BM) || !make_map(&mb, p.b, p.k, p.n, p.ldb, 16))
        return launch_dmma<Cfg128>(s, p0);
    uint32_t* flags = nullptr;
    double* park = nullptr;
    kw_status st = split_scratch(s, G, 4 + static_cast<size_t>(VG) * Cfg::CONSUMERS,
                                 static_cast<size_t>(VG) * Cfg::CONSUMERS * Cfg::MT * Cfg::NT * 32 * sizeof(double2), &flags,
                                 &park);
    if (st != KW_OK)
        return st;
    p.ready = flags;
    p.partial = park;
#if defined(KW_SPLIT_TRACE)
    p.tile_list = static_cast<const int4*>(g_split_trace.load(std::memory_order_relaxed)); // trace or null
#else
    p.tile_list = nullptr;
#endif
    p.panel_rows = dgemm_group();
    static const long long dp_env = [] { // KW_SPLIT_DP_TILES: data-parallel tile count override (sweeps)
        const char* e = std::getenv("KW_SPLIT_DP_TILES");
        return e ? std::atoll(e) : -1ll;
    }();
    p.npr = static_cast<int>(dp_env);
    st = ensure_smem(reinterpret_cast<const void*>(dgemm_tma_kernel<Cfg, false, true>), Cfg::SMEM,
                     "dgemm: cudaFuncSetAttribute");
    if (st != KW_OK)
        return st;
    if (cudaError_t e = launch_tma_kernel<Cfg, false, true>(static_cast<unsigned>(G), s, ma, mb, p, true))
        return kw::cuda_fail("dgemm (split): launch", e);
    kw::g_launches.fetch_add(1, std::memory_order_relaxed);
    return KW_OK;
}

// One k-tile range [kt0, kt1) of every tile of a resident product (KRANGE), parking to /
// reloading from `park` (dgemm_krange_park_bytes).
template <class Cfg>
kw_status launch_krange(cudaStream_t s, const GemmParams& p0, int kt0, int kt1, double* park)
{
    GemmParams p = p0;
    p.tiles_m = static_cast<int>(kw::ceil_div(p.m, Cfg::BM));
    p.tiles_n = static_cast<int>(kw::ceil_div(p.n, Cfg::BN));
    const long long tiles = static_cast<long long>(p.tiles_m) * p.tiles_n;
    if (tiles > INT_MAX)
        return kw::usage("dgemm: problem too large for the tile grid");
    if (!tma_eligible(p))
        return kw::usage("dgemm (k-range): operands not TMA-addressable");
    CUtensorMap ma, mb;
    if (!make_map(&ma, p.a, p.m, p.k, p.lda, Cfg::BM) || !make_map(&mb, p.b, p.k, p.n, p.ldb, 16))
        return kw::usage("dgemm (k-range): tensor map encoding failed");
    const kw_status st = ensure_smem(reinterpret_cast<const void*>(dgemm_tma_kernel<Cfg, false, false, true>),
                                     Cfg::SMEM, "dgemm: cudaFuncSetAttribute");
    if (st != KW_OK)
        return st;
    p.npr = kt0;
    p.npc = kt1;
    p.partial = park;
    p.panel_rows = dgemm_group();
    p.panel_cols = 0; // not split-k (launch_splitk)
    const long long resident = static_cast<long long>(sm_count()) * Cfg::MIN_BLOCKS;
    if (cudaError_t e = launch_tma_kernel<Cfg, false, false, true>(static_cast<unsigned>(tiles), s, ma, mb, p,
                                                                   tiles >= resident))
        return kw::cuda_fail("dgemm (k-range): launch", e);
    kw::g_launches.fetch_add(1, std::memory_order_relaxed);
    return KW_OK;
}

// Split-k park (per stream, the SplitScratch entry's park buffer; no tickets or flags involved).
kw_status splitk_park(cudaStream_t s, size_t bytes, double** park)
{
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(g_split_mu);
    SplitScratch* sc = nullptr;
    for (SplitScratch* x : g_split)
        if (x->device == dev && x->stream == s)
            sc = x;
    if (!sc) {
        sc = new SplitScratch;
        sc->device = dev;
        sc->stream = s;
        g_split.push_back(sc);
    }
    if (sc->park_bytes < bytes) {
        cudaStreamSynchronize(s); // earlier launches on this stream may still use the old park
        cudaFree(sc->park);
        sc->park = nullptr;
        sc->park_bytes = 0;
        if (cudaError_t e = cudaMalloc(&sc->park, bytes))
            return kw::cuda_fail("dgemm split-k: park scratch", e);
        sc->park_bytes = bytes;
    }
    *park = sc->park;
    return KW_OK;
}

// Split-k reduction: C = alpha * (P_0 + P_1 + ... + P_{S-1}) + beta * C over the S partial
// chains of launch_splitk, added in slice order (deterministic); one CTA per tile, one thread per
// (consumer warp, lane) fragment set of the park layout, the main kernel's epilogue arithmetic.
template <class Cfg>
__global__ void __launch_bounds__(Cfg::CONSUMERS * 32) splitk_reduce_kernel(GemmParams p, int slices)
{
    const int tile = blockIdx.x;
    const int tr = tile / p.tiles_n, tc = tile - tr * p.tiles_n;
    const int lw = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int wm = (lw / Cfg::WARPS_N) * Cfg::WM, wn = (lw % Cfg::WARPS_N) * Cfg::WN;
    const size_t stride = static_cast<size_t>(p.tiles_m) * p.tiles_n * Cfg::CONSUMERS * (Cfg::MT * Cfg::NT) * 32;
    const double2* base = reinterpret_cast<const double2*>(p.partial) +
                          (static_cast<size_t>(tile) * Cfg::CONSUMERS + lw) * (Cfg::MT * Cfg::NT) * 32 + lane;
    const bool c_vec = (p.ldc % 2 == 0) && (reinterpret_cast<uintptr_t>(p.c) % 16 == 0);
    for (int i = 0; i < Cfg::MT; ++i) {
        const int row = tr * Cfg::BM + wm + i * 8 + g;
        if (row >= p.m)
            continue;
        double* crow = p.c + static_cast<size_t>(row) * p.ldc;
        for (int j = 0; j < Cfg::NT; ++j) {
            const int col = tc * Cfg::BN + wn + j * 8 + 2 * t;
            if (col >= p.n)
                continue;
            const double2* src = base + (i * Cfg::NT + j) * 32;
            double2 acc = __ldcs(src);
            for (int sl = 1; sl < slices; ++sl) {
                const double2 v = __ldcs(src + sl * stride);
                acc.x = __dadd_rn(acc.x, v.x);
                acc.y = __dadd_rn(acc.y, v.y);
            }
            double2 old;
            if (c_vec && col + 1 < p.n)
                old = *reinterpret_cast<const double2*>(crow + col);
            else {
                old.x = crow[col];
                old.y = col + 1 < p.n ? crow[col + 1] : 0.0;
            }
            const double x = __dadd_rn(__dmul_rn(p.alpha, acc.x), __dmul_rn(p.beta, old.x));
            const double y = __dadd_rn(__dmul_rn(p.alpha, acc.y), __dmul_rn(p.beta, old.y));
            if (c_vec && col + 1 < p.n)
                *reinterpret_cast<double2*>(crow + col) = make_double2(x, y);
            else {
                crow[col] = x;
                if (col + 1 < p.n)
                    crow[col + 1] = y;
            }
        }
    }
}

// Split-k for small outputs with long k (fewer 64 x 64 tiles than SMs): the one-CTA-per-tile
// chain leaves most SMs idle (512 x 512 x 16384: 64 tiles, 12.3 TFLOP/s) and the SPLIT walk
// cannot help (a tile's chain is split at most once). Here the k-tiles are cut into S slices,
// one k-range launch runs every (tile, slice) as an independent chain from zero (grid tiles x
// S, parked per slice), and splitk_reduce_kernel adds the S partials in slice order and runs the
// epilogue. Deterministic, within the same (K+4)u bound, but NOT the bits of the one-CTA chain:
// this is the one resident path whose bits depend on the configuration.
template <class Cfg>
kw_status launch_splitk(cudaStream_t s, const GemmParams& p0)
{
    GemmParams p = p0;
    p.tiles_m = static_cast<int>(kw::ceil_div(p.m, Cfg::BM));
    p.tiles_n = static_cast<int>(kw::ceil_div(p.n, Cfg::BN));
    const long long tiles = static_cast<long long>(p.tiles_m) * p.tiles_n;
    const long long ktiles = kw::ceil_div(p.k, Cfg::BK);
    const long long resident = static_cast<long long>(sm_count()) * Cfg::MIN_BLOCKS;
    // Slices: as many as keep every SM at <= 2 CTAs (tiles * S <= 2 * SMs; 16..24 k-tiles per
    // slice at least/most apart): measured best or within 5 % of the best S on 512^2 x 16384
    // (S = 4: 27.6 TFLOP/s), 768^2 x 8192 (2: 31.7), 512^2 x 4096 (4: 22.3), 512^2 x 2048 (4:
    // 17.4 vs 11.6 data-parallel) — profiles/dgemm_splitk_r02.txt. KW_SPLITK_SLICES overrides.
    static const long long env_s = [] {
        const char* e = std::getenv("KW_SPLITK_SLICES");
        return e ? std::atoll(e) : 0ll;
    }();
    long long S = env_s > 0 ? env_s
                            : std::min<long long>(24, 2 * static_cast<long long>(sm_count()) / std::max<long long>(tiles, 1));
    S = std::max<long long>(2, std::min<long long>(S, ktiles / 16));
    const long long kts = S > 1 ? kw::ceil_div(ktiles, S) : ktiles;
    S = kw::ceil_div(ktiles, kts);
    if (S < 2 || tiles > INT_MAX || !tma_eligible(p))
        return launch_tma<Tma64x64x3p>(s, p0);
    CUtensorMap ma, mb;
    if (!make_map(&ma, p.a, p.m, p.k, p.lda, Cfg::BM) || !make_map(&mb, p.b, p.k, p.n, p.ldb, 16))
        return launch_tma<Tma64x64x3p>(s, p0);
    double* park = nullptr;
    kw_status st = splitk_park(s, static_cast<size_t>(S) * tiles * Cfg::CONSUMERS * Cfg::MT * Cfg::NT * 32 * sizeof(double2),
                               &park);
    if (st != KW_OK)
        return st;
    st = ensure_smem(reinterpret_cast<const void*>(dgemm_tma_kernel<Cfg, false, false, true>), Cfg::SMEM,
                     "dgemm: cudaFuncSetAttribute");
    if (st != KW_OK)
        return st;
    p.npr = p.npc = 0;
    p.panel_cols = static_cast<int>(kts); // > 0: split-k slices (dgemm_tma_kernel KRANGE)
    p.partial = park;
    p.panel_rows = dgemm_group();
    if (cudaError_t e = launch_tma_kernel<Cfg, false, false, true>(static_cast<unsigned>(tiles), s, ma, mb, p, false,
                                                                   static_cast<unsigned>(S)))
        return kw::cuda_fail("dgemm (split-k): launch", e);
    splitk_reduce_kernel<Cfg><<<static_cast<unsigned>(tiles), Cfg::CONSUMERS * 32, 0, s>>>(p, static_cast<int>(S));
    if (cudaError_t e = cudaGetLastError())
        return kw::cuda_fail("dgemm (split-k): reduction launch", e);
    kw::g_launches.fetch_add(2, std::memory_order_relaxed);
    return KW_OK;
}

struct CfgInfo {
    int bm, bn, bk, threads, stages;
    kw_status (*launch)(cudaStream_t, const GemmParams&);
};

const CfgInfo kCfgs[] = {
    {Cfg128::BM, Cfg128::BN, Cfg128::BK, Cfg128::THREADS, Cfg128::STAGES, launch_dmma<Cfg128>},
    {Cfg128k32::BM, Cfg128k32::BN, Cfg128k32::BK, Cfg128k32::THREADS, Cfg128k32::STAGES, launch_dmma<Cfg128k32>},
    {Cfg128w16::BM, Cfg128w16::BN, Cfg128w16::BK, Cfg128w16::THREADS, Cfg128w16::STAGES, launch_dmma<Cfg128w16>},
    {Cfg128w16k32::BM, Cfg128w16k32::BN, Cfg128w16k32::BK, Cfg128w16k32::THREADS, Cfg128w16k32::STAGES,
     launch_dmma<Cfg128w16k32>},
    {Cfg64::BM, Cfg64::BN, Cfg64::BK, Cfg64::THREADS, Cfg64::STAGES, launch_dmma<Cfg64>},
    {Cfg128x64::BM, Cfg128x64::BN, Cfg128x64::BK, Cfg128x64::THREADS, Cfg128x64::STAGES, launch_dmma<Cfg128x64>},
    {Cfg64x128::BM, Cfg64x128::BN, Cfg64x128::BK, Cfg64x128::THREADS, Cfg64x128::STAGES, launch_dmma<Cfg64x128>},
    {Tma128::BM, Tma128::BN, Tma128::BK, Tma128::THREADS, Tma128::STAGES, launch_tma<Tma128>},
    {Tma128s4::BM, Tma128s4::BN, Tma128s4::BK, Tma128s4::THREADS, Tma128s4::STAGES, launch_tma<Tma128s4>},
    {Tma64x128::BM, Tma64x128::BN, Tma64x128::BK, Tma64x128::THREADS, Tma64x128::STAGES, launch_tma<Tma64x128>},
    {Tma128x64::BM, Tma128x64::BN, Tma128x64::BK, Tma128x64::THREADS, Tma128x64::STAGES, launch_tma<Tma128x64>},
    {Tma128s7::BM, Tma128s7::BN, Tma128s7::BK, Tma128s7::THREADS, Tma128s7::STAGES, launch_tma<Tma128s7>},
    {Tma128x64x2::BM, Tma128x64x2::BN, Tma128x64x2::BK, Tma128x64x2::THREADS, Tma128x64x2::STAGES,
     launch_tma<Tma128x64x2>},
    {Tma64x128x2::BM, Tma64x128x2::BN, Tma64x128x2::BK, Tma64x128x2::THREADS, Tma64x128x2::STAGES,
     launch_tma<Tma64x128x2>},
    {Tma128p::BM, Tma128p::BN, Tma128p::BK, Tma128p::THREADS, Tma128p::STAGES, launch_tma<Tma128p>},
    {Tma128p::BM, Tma128p::BN, Tma128p::BK, Tma128p::THREADS, Tma128p::STAGES, launch_tma<Tma128p, true>}, // 15: persistent
    {Tma64x128x2p::BM, Tma64x128x2p::BN, Tma64x128x2p::BK, Tma64x128x2p::THREADS, Tma64x128x2p::STAGES,
     launch_tma<Tma64x128x2p>},
    {Tma64x64x3p::BM, Tma64x64x3p::BN, Tma64x64x3p::BK, Tma64x64x3p::THREADS, Tma64x64x3p::STAGES,
     launch_tma<Tma64x64x3p>},
    {Split64w8::BM, Split64w8::BN, Split64w8::BK, Split64w8::THREADS, Split64w8::STAGES, launch_split<Split64w8>},
    {Split64w4::BM, Split64w4::BN, Split64w4::BK, Split64w4::THREADS, Split64w4::STAGES, launch_split<Split64w4>},
    {Split64x128w8::BM, Split64x128w8::BN, Split64x128w8::BK, Split64x128w8::THREADS, Split64x128w8::STAGES,
     launch_split<Split64x128w8>},
    {Tma64x128x2p::BM, Tma64x128x2p::BN, Tma64x128x2p::BK, Tma64x128x2p::THREADS, Tma64x128x2p::STAGES,
     launch_split<Tma64x128x2p>}, // 21: SPLIT of config 16 (two CTAs per SM)
    {Tma64x64x3p::BM, Tma64x64x3p::BN, Tma64x64x3p::BK, Tma64x64x3p::THREADS, Tma64x64x3p::STAGES,
     launch_split<Tma64x64x3p>}, // 22: SPLIT of config 17 (three CTAs per SM)
    {Split64w8t::BM, Split64w8t::BN, Split64w8t::BK, Split64w8t::THREADS, Split64w8t::STAGES,
     launch_split<Split64w8t>},
    {Tma128p::BM, Tma128p::BN, Tma128p::BK, Tma128p::THREADS, Tma128p::STAGES,
     launch_split<Tma128p>}, // 24: SPLIT of config 14 (128 x 128, 8 consumers of 64 x 32, 1 CTA/SM)
    {Pair64x128::BM, Pair64x128::BN, Pair64x128::BK, Pair64x128::THREADS, Pair64x128::STAGES,
     launch_split<Pair64x128>}, // 25
    {Pair64x128::BM, Pair64x128::BN, Pair64x128::BK, Pair64x128::THREADS, Pair64x128::STAGES,
     launch_tma<Pair64x128>}, // 26
    {Tma64x64x3p::BM, Tma64x64x3p::BN, Tma64x64x3p::BK, Tma64x64x3p::THREADS, Tma64x64x3p::STAGES,
     launch_splitk<Tma64x64x3p>}, // 27: split-k over config 17 (NOT bitwise-interchangeable)
    {Tma32p::BM, Tma32p::BN, Tma32p::BK, Tma32p::THREADS, Tma32p::STAGES, launch_tma<Tma32p>},         // 28
    {Tma32x64p::BM, Tma32x64p::BN, Tma32x64p::BK, Tma32x64p::THREADS, Tma32x64p::STAGES, launch_tma<Tma32x64p>}, // 29
};
constexpr int kNumCfgs = sizeof(kCfgs) / sizeof(kCfgs[0]);
// Tile choice for the GPU back-end. The tile work division (gemmTiledWorkDiv) is the coverage
// contract; the kernel picks its CTA tile among the paired-k-map TMA configurations, which feed
// every output element the identical DMMA sequence (test_paired_configs_are_bitwise_
// interchangeable) — so the choice never changes a bit, and row panels, column panels and row
// shards of one product still reproduce the single launch exactly.
//   16: 64x128 tile, 2 CTAs/SM (best from ~1536 up: 35.4 TFLOP/s at 8192^3, 34.7 at 4096^3)
//   17: 64x64 tile, 3 CTAs/SM  (best for small outputs: 26.4 at 1024^3, 33.0 at 2048^3)
// Model: the busiest SM's output count, ceil(tiles / SMs) * tile area; take 17 when that is >3%
// lower, or when 16 would not give every SM a tile (1 CTA per SM under-feeds the DMMA pipe), or
// for short k (< 1408): short k-loops make the per-tile epilogue a larger share, which three
// co-resident CTAs hide better (8192 x 8192 x 256: 33.1 vs 32.0 TFLOP/s; x 1024: 35.3 vs 34.9;
// 3000 x 5000 x 700: 32.9 vs 32.1; at k = 1536 16 leads again, 4096^2 x 1536: 35.06 vs 34.96 —
// profiles/dgemm_rect_r02.txt).
// Fewer 64 x 64 tiles than SMs: smaller tiles of the same paired k-map (bits unchanged) — 32 x 64
// (29, two CTAs/SM) from 1.5 of its tiles per SM, else 32 x 32 (28, three CTAs/SM): 512^2 x
// 16384 12.3 -> 27.4 TFLOP/s (28), 768^2 x 8192 27.4 -> 33.0 (29), 512^2 x 2048 11.6 -> 24.9 (28;
// cuBLAS 22.8) — profiles/dgemm_small_tiles_r02.txt.
constexpr int kCfgWide = 16, kCfgSmall = 17, kCfgTiny = 28, kCfgTinyWide = 29;
constexpr int kShortK = 1408;

int pick_config(const GemmParams& p)
{
    const long long sms = sm_count();
    const long long rows = (p.m + 63) / 64;
    const long long t16 = rows * ((p.n + 127) / 128), t17 = rows * ((p.n + 63) / 64);
    if (t17 < sms) {
        const long long t29 = ((p.m + 31) / 32) * ((p.n + 63) / 64);
        return 2 * t29 >= 3 * sms ? kCfgTinyWide : kCfgTiny;
    }
    const long long load16 = (t16 + sms - 1) / sms * 8192, load17 = (t17 + sms - 1) / sms * 4096;
    const bool small =
        t16 <= sms || p.k < kShortK || static_cast<double>(load17) < 0.97 * static_cast<double>(load16);
    return small ? kCfgSmall : kCfgWide;
}

// Resident launches add the SPLIT configurations (one CTA per SM over equal (tile, k-tile)
// ranges — same paired DMMA sequence, so again no bit changes) where both data-parallel grids
// quantise badly: the busiest SM of the better of 16 / 17 carries more than 1/0.93 of the mean
// output (1024^3: 2 of 1.73 tiles, 0.865 -> split 18 at 30.8 vs 27.6 TFLOP/s). By tiles of
// 64 x 128 per SM: below 1, split 18 (64 x 64, 8 warps of 32 x 16, C prefetched into registers);
// 1 to 2.5, split 20 (64 x 128, 8 warps of 32 x 32; 1280^3 32.6 vs 18: 32.2); above, the
// two-group split 25 (1792^3 33.9 vs 20: 33.7). profiles/dgemm_prefetch_ab_r02.txt.
constexpr int kCfgSplit64 = 18, kCfgSplit128 = 20, kCfgSplitPair = 25, kCfgSplitK = 27;
// Split-k (config 27) below a full wave of 64 x 64 tiles with a long k — opt-in (KW_DGEMM_SPLITK=1):
// it is the one configuration whose bits differ from the one-CTA chain, and by default every
// path (resident, host-staged, streamed, row-sharded) gives the same bits, the GPU analogue of
// the reference's cross-backend determinism (acceptance criterion 01). See launch_splitk.
constexpr long long kSplitKMinKtiles = 64;
bool splitk_default()
{
    static const bool on = [] {
        const char* e = std::getenv("KW_DGEMM_SPLITK");
        return e && e[0] == '1';
    }();
    return on;
}
int pick_resident(const GemmParams& p)
{
    const double sms = sm_count();
    const long long rows = (p.m + 63) / 64;
    const long long t16 = rows * ((p.n + 127) / 128), t17 = rows * ((p.n + 63) / 64);
    const double ideal = static_cast<double>(p.m) * p.n / sms;
    const double q16 = ideal / (std::ceil(t16 / sms) * 8192.0), q17 = ideal / (std::ceil(t17 / sms) * 4096.0);
    const long long ktiles = (p.k + 15) / 16;
    const long long t28 = ((p.m + 31) / 32) * ((p.n + 31) / 32);
    if (splitk_default() && t28 < static_cast<long long>(sms) && ktiles >= kSplitKMinKtiles && tma_eligible(p))
        return kCfgSplitK;
    if (std::max(q16, q17) < 0.93 && t17 >= static_cast<long long>(sms) && ktiles >= 2 && tma_eligible(p))
        return 2 * t16 >= 5 * static_cast<long long>(sms) ? kCfgSplitPair
               : t16 >= static_cast<long long>(sms)       ? kCfgSplit128
                                                          : kCfgSplit64;
    // Mid-size outputs (2 to 16 tiles of 64 x 128 per consumer group) whose 64 x 128 grid leaves a
    // partial last wave: the two-group SPLIT config (config 16's geometry twice in one CTA, equal
    // k-tile ranges) — 2048^3 34.3 vs 34.0, 3072^3 35.0 vs 34.4, 3584^3 35.1 vs 34.2, 6144^3
    // 35.4 vs 35.1 TFLOP/s; where config 16's waves come out whole (4096^3: 6.92 of 7) or are many
    // (>= 7168^3) the data-parallel grid stays ahead (profiles/dgemm_split_sweep_r02.txt).
    // (Not for k < 1536 where config 17's grid quantises well: 2304^2 x 768 17: 33.2 vs 25: 32.0,
    // 6144^2 x 768 34.8 vs 33.8, 6144^2 x 1280 35.1 vs 34.6, 3000 x 5000 x 1024 33.4 vs 33.1.)
    const bool short_k_17 = p.k < 1536 && q17 >= 0.95;
    if (t16 >= 2 * static_cast<long long>(sms) && t16 <= 32 * static_cast<long long>(sms) && q16 < 0.985 &&
        !short_k_17 && ktiles >= 2 && tma_eligible(p))
        return kCfgSplitPair;
    return pick_config(p);
}


GemmParams make_params(size_t m, size_t n, size_t k, double alpha, const double* A, size_t lda, const double* B,
                       size_t ldb, double beta, double* C, size_t ldc)
{
    GemmParams p;
    p.m = static_cast<int>(m);
    p.n = static_cast<int>(n);
    p.k = static_cast<int>(k);
    p.alpha = alpha;
    p.beta = beta;
    p.a = A;
    p.lda = static_cast<long long>(lda);
    p.b = B;
    p.ldb = static_cast<long long>(ldb);
    p.c = C;
    p.ldc = static_cast<long long>(ldc);
    p.tiles_m = p.tiles_n = 0;
    p.tile_list = nullptr;
    p.ready = nullptr;
    p.partial = nullptr;
    p.panel_rows = p.panel_cols = 1;
    p.npr = p.npc = 0;
    return p;
}

size_t round2(size_t v) { return (v + 1) & ~static_cast<size_t>(1); }

} // namespace

namespace kw::gemm {
// The interface the host-operand schedules (kw_dgemm_e2e.cu) and the row-sharded driver use.
GemmParams make_params(size_t m, size_t n, size_t k, double alpha, const double* A, size_t lda, const double* B,
                       size_t ldb, double beta, double* C, size_t ldc)
{
    return ::make_params(m, n, k, alpha, A, lda, B, ldb, beta, C, ldc);
}
size_t round2(size_t v) { return ::round2(v); }
// Data-parallel choices only (16 / 17): for callers that overlap consecutive launches on two
// streams (the host-staged row-panel schedule), where one-CTA-per-SM SPLIT grids could not overlap.
kw_status launch_tiled_dp(cudaStream_t s, int tile, const GemmParams& p)
{
    return kCfgs[tile == 64 ? kCfgSmall : pick_config(p)].launch(s, p);
}
kw_status launch_tiled(cudaStream_t s, int tile, const GemmParams& p)
{
    const int cfg = tile == 64 ? kCfgSmall : pick_resident(p);
    static const bool log = std::getenv("KW_DGEMM_LOG") != nullptr; // tile-choice trace (debugging)
    if (log)
        std::fprintf(stderr, "[kw dgemm] %d x %d x %d tile %d -> config %d (tma %d)\n", p.m, p.n, p.k, tile, cfg,
                     static_cast<int>(tma_eligible(p)));
    return kCfgs[cfg].launch(s, p);
}
bool tma_eligible(const GemmParams& p)
{
    return p.k > 0 && (p.lda * 8) % 16 == 0 && (p.ldb * 8) % 16 == 0 && reinterpret_cast<uintptr_t>(p.a) % 16 == 0 &&
           reinterpret_cast<uintptr_t>(p.b) % 16 == 0 && encode_fn() != nullptr;
}
int streamed_config(int tile, const GemmParams& p) { return tile == 64 ? kCfgSmall : pick_config(p); }
StreamedShape streamed_shape(int cfg)
{
    return cfg == kCfgWide ? StreamedShape{Tma64x128x2p::BM, Tma64x128x2p::BN, Tma64x128x2p::CONSUMERS}
                           : StreamedShape{Tma64x64x3p::BM, Tma64x64x3p::BN, Tma64x64x3p::CONSUMERS};
}
int streamed_grid(int cfg, const GemmParams& p)
{
    // launch_tma<.., PERSISTENT = true, ..>'s grid: min(tiles, resident CTAs)
    const StreamedShape sh = streamed_shape(cfg);
    const long long tiles = static_cast<long long>(kw::ceil_div(p.m, sh.bm)) * kw::ceil_div(p.n, sh.bn);
    const long long resident =
        static_cast<long long>(sm_count()) * (cfg == kCfgWide ? Tma64x128x2p::MIN_BLOCKS : Tma64x64x3p::MIN_BLOCKS);
    return static_cast<int>(tiles > resident ? resident : tiles);
}
kw_status launch_streamed(cudaStream_t s, int cfg, const GemmParams& p)
{
    return cfg == kCfgWide ? launch_tma<Tma64x128x2p, true, true>(s, p) : launch_tma<Tma64x64x3p, true, true>(s, p);
}
} // namespace kw::gemm

namespace kw {
uint32_t split_take_abort(cudaStream_t s)
{
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(g_split_mu);
    for (SplitScratch* x : g_split)
        if (x->device == dev && x->stream == s && x->abort_host) {
            const uint32_t v = *reinterpret_cast<volatile uint32_t*>(x->abort_host);
            if (v) {
                // A timed-out wait leaves head flags raised that no tail consumed: clear the
                // ticket and every flag (not the abort pointer, words 2-3) before the next launch.
                x->abort_host[0] = 0;
                cudaStreamSynchronize(s);
                cudaMemsetAsync(x->flags, 0, 8, s);
                if (x->flag_words > 4)
                    cudaMemsetAsync(x->flags + 4, 0, (x->flag_words - 4) * sizeof(uint32_t), s);
                cudaStreamSynchronize(s);
            }
            return v;
        }
    return 0;
}

void split_release(cudaStream_t s)
{
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(g_split_mu);
    for (size_t i = 0; i < g_split.size(); ++i) {
        SplitScratch* x = g_split[i];
        if (x->device == dev && x->stream == s) {
            cudaStreamSynchronize(s);
            cudaFree(x->flags);
            cudaFree(x->park);
            cudaFreeHost(x->abort_host);
            delete x;
            g_split.erase(g_split.begin() + static_cast<long>(i));
            return;
        }
    }
}

// Used by the row-sharded driver (kw_comm.cu).
kw_status dgemm_device(cudaStream_t s, int tile, size_t m, size_t n, size_t k, double alpha, const double* A,
                       size_t lda, const double* B, size_t ldb, double beta, double* C, size_t ldc)
{
    if (m == 0 || n == 0)
        return KW_OK;
    return launch_tiled(s, tile, make_params(m, n, k, alpha, A, lda, B, ldb, beta, C, ldc));
}

// The data-parallel configuration for the whole m x n x k problem (row-sharded: every panel
// launch of a rank uses it, so panel grids on the two compute streams co-reside evenly and fill
// each other's tails; one-CTA-per-SM SPLIT grids cannot overlap — measured 33.6 vs 34.6 TFLOP/s
// for a 2048-row rank, profiles/rowshard_rank_probe_r02.txt).
int dgemm_pick(size_t m, size_t n, size_t k)
{
    return pick_config(make_params(m, n, k, 1.0, nullptr, k, nullptr, n, 0.0, nullptr, n));
}

// Whether the k-range launches can run on these operands (TMA-addressable A and B).
bool dgemm_krange_ok(size_t m, size_t n, size_t k, const double* A, size_t lda, const double* B, size_t ldb)
{
    return m > 0 && n > 0 && tma_eligible(make_params(m, n, k, 1.0, A, lda, B, ldb, 0.0, nullptr, n));
}

// k-range passes for the row-sharded k-slab schedule: config 16 for its own pick, 17 (64 x 64)
// for every other data-parallel pick (same bits).
size_t dgemm_krange_park_bytes(int cfg, size_t m, size_t n)
{
    const size_t bm = 64, bn = cfg == kCfgWide ? 128 : 64;
    return kw::ceil_div(m, bm) * bm * kw::ceil_div(n, bn) * bn * sizeof(double);
}

kw_status dgemm_device_krange(cudaStream_t s, int cfg, size_t m, size_t n, size_t k, double alpha, const double* A,
                              size_t lda, const double* B, size_t ldb, double beta, double* C, size_t ldc, int kt0,
                              int kt1, double* park)
{
    if (m == 0 || n == 0)
        return KW_OK;
    const GemmParams p = make_params(m, n, k, alpha, A, lda, B, ldb, beta, C, ldc);
    return cfg == kCfgWide ? launch_krange<Tma64x128x2p>(s, p, kt0, kt1, park)
                           : launch_krange<Tma64x64x3p>(s, p, kt0, kt1, park);
}

kw_status dgemm_device_cfg(cudaStream_t s, int cfg, size_t m, size_t n, size_t k, double alpha, const double* A,
                           size_t lda, const double* B, size_t ldb, double beta, double* C, size_t ldc)
{
    if (m == 0 || n == 0)
        return KW_OK;
    if (cfg < 0 || cfg >= kNumCfgs)
        return kw::usage("dgemm: configuration index out of range");
    return kCfgs[cfg].launch(s, make_params(m, n, k, alpha, A, lda, B, ldb, beta, C, ldc));
}
} // namespace kw

namespace {
// The device-only entry points (bitwise, naive, with_config): every operand is device memory on
// the queue's own device — a buffer of another GPU (no peer mapping) would fault the context.
kw_status device_operands(const kw::Queue* q, const char* what, size_t k, const double* A, const double* B,
                          const double* C)
{
    const double* ops[3] = {C, A, B};
    for (int i = 0; i < (k > 0 ? 3 : 1); ++i) {
        int d = -1;
        if (kw::pointer_kind(ops[i], &d) != KW_MEM_DEVICE)
            return kw::usage(std::string(what) + ": operands must be device buffers");
        if (d != q->device)
            return kw::usage(std::string(what) + ": buffer lives on a different device than the queue");
    }
    return KW_OK;
}
} // namespace

extern "C" {

kw_status kw_dgemm_default_workdiv(size_t m, size_t n, size_t tile, kw_workdiv* out)
{
    if (!out)
        return kw::usage("kw_dgemm_default_workdiv: null output");
    if (tile == 0)
        tile = 128;
    kw_workdiv wd = {};
    wd.dim = 2;
    for (int k = 0; k < 3; ++k)
        wd.blocks[k] = wd.threads[k] = wd.elems[k] = 1;
    if (tile == 128) {
        wd.threads[0] = 16;
        wd.threads[1] = 16;
        wd.elems[0] = 8;
        wd.elems[1] = 8;
    }
    else if (tile == 64) {
        wd.threads[0] = 8;
        wd.threads[1] = 16;
        wd.elems[0] = 8;
        wd.elems[1] = 4;
    }
    else {
        return kw::usage("gemmTiledWorkDiv: GPU tile edge must be 64 or 128");
    }
    wd.blocks[0] = kw::ceil_div(m == 0 ? 1 : m, tile);
    wd.blocks[1] = kw::ceil_div(n == 0 ? 1 : n, tile);
    *out = wd;
    return KW_OK;
}

kw_status kw_dgemm(kw_queue qh, const kw_workdiv* wd, size_t m, size_t n, size_t k, double alpha, const double* A,
                   size_t lda, const double* B, size_t ldb, double beta, double* C, size_t ldc)
{
    KW_CHECK_QUEUE(qh);
    KW_ENQUEUE_LOCK(qh);
    KW_NVTX("kw dgemm");
    auto* q = reinterpret_cast<kw::Queue*>(qh);
    kw_status st = validate_gemm(m, n, k, A, lda, B, ldb, C, ldc);
    if (st != KW_OK)
        return st;
    int tile = 128;
    st = tile_from_wd(wd, m, n, &tile);
    if (st != KW_OK)
        return st;
    if (m == 0 || n == 0)
        return KW_OK;
    kw::DeviceGuard g(q->device);
    int da = -1, db = -1, dc = -1;
    const bool a_dev = k == 0 || kw::pointer_kind(A, &da) == KW_MEM_DEVICE;
    const bool b_dev = k == 0 || kw::pointer_kind(B, &db) == KW_MEM_DEVICE;
    const bool c_dev = kw::pointer_kind(C, &dc) == KW_MEM_DEVICE;
    if ((da >= 0 && a_dev && da != q->device) || (db >= 0 && b_dev && db != q->device) ||
        (c_dev && dc != q->device))
        return kw::usage("dgemm: buffer lives on a different device than the queue");
    if (a_dev && b_dev && c_dev) {
        st = launch_tiled(q->stream, tile, make_params(m, n, k, alpha, A, lda, B, ldb, beta, C, ldc));
        if (st != KW_OK)
            return kw::task_fail(q, kw::last_error());
        return kw::after_enqueue(q, "dgemm");
    }
    if (!a_dev && !b_dev && !c_dev && kw::pointer_kind(A, nullptr) == KW_MEM_PINNED &&
        kw::pointer_kind(B, nullptr) == KW_MEM_PINNED && kw::pointer_kind(C, nullptr) == KW_MEM_PINNED) {
        bool used = false;
        st = kw::gemm::dgemm_streamed(q, tile, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, &used);
        if (st != KW_OK || used)
            return st;
    }
    return kw::gemm::dgemm_staged(q, tile, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, a_dev, b_dev, c_dev);
}


kw_status kw_dgemm_bitwise(kw_queue qh, const kw_workdiv* wd, size_t m, size_t n, size_t k, double alpha,
                           const double* A, size_t lda, const double* B, size_t ldb, double beta, double* C, size_t ldc)
{
    KW_CHECK_QUEUE(qh);
    KW_ENQUEUE_LOCK(qh);
    KW_NVTX("kw dgemm (bit-exact mode)");
    auto* q = reinterpret_cast<kw::Queue*>(qh);
    kw_status st = validate_gemm(m, n, k, A, lda, B, ldb, C, ldc);
    if (st != KW_OK)
        return st;
    if (wd != nullptr) {
        if (wd->dim != 2)
            return kw::usage("dgemm_bitwise: the tiled kernel runs on a 2-D (rows, cols) work division");
        if (wd->threads[0] * wd->elems[0] != 128 || wd->threads[1] * wd->elems[1] != 128 ||
            wd->threads[0] * wd->threads[1] != 256)
            return kw::usage("dgemm_bitwise: the bitwise tiled kernel runs 128x128 tiles of 256 threads "
                             "(gemmTiledWorkDiv(GpuCudaRt, m, n, 128))");
        if (wd->blocks[0] * 128 < m || wd->blocks[1] * 128 < n)
            return kw::usage("dgemm: work division does not cover the m x n output");
    }
    if (m == 0 || n == 0)
        return KW_OK;
    kw::DeviceGuard g(q->device);
    st = device_operands(q, "dgemm_bitwise", k, A, B, C);
    if (st != KW_OK)
        return st;
    st = launch_bitwise(q->stream, make_params(m, n, k, alpha, A, lda, B, ldb, beta, C, ldc));
    if (st != KW_OK)
        return kw::task_fail(q, kw::last_error());
    return kw::after_enqueue(q, "dgemm_bitwise");
}

int kw_dgemm_config_count(void) { return kNumCfgs; }

kw_status kw_dgemm_split_trace(void* device_buffer)
{
    g_split_trace.store(device_buffer, std::memory_order_relaxed);
    return KW_OK;
}

kw_status kw_dgemm_split_plan(long long tiles, long long ktiles, long long ctas, long long cta, long long dp_tiles,
                              int out[11])
{
    if (!out || tiles < ctas || ctas < 1 || ktiles < 1 || cta < 0 || cta >= ctas)
        return kw::usage("kw_dgemm_split_plan: needs tiles >= ctas >= 1, ktiles >= 1, 0 <= cta < ctas");
    const SplitRange r = split_range(tiles, ktiles, ctas, cta, dp_tiles);
    const int v[11] = {r.ndp, r.dp0, r.dp_step, r.head, r.nfull, r.tail, r.t_head, r.x_head, r.t_full0, r.t_tail,
                       r.x_tail};
    std::memcpy(out, v, sizeof(v));
    return KW_OK;
}

kw_status kw_dgemm_config_info(int cfg, int info[5])
{
    if (cfg < 0 || cfg >= kNumCfgs || !info)
        return kw::usage("dgemm config index out of range");
    info[0] = kCfgs[cfg].bm;
    info[1] = kCfgs[cfg].bn;
    info[2] = kCfgs[cfg].bk;
    info[3] = kCfgs[cfg].threads;
    info[4] = kCfgs[cfg].stages;
    return KW_OK;
}

kw_status kw_dgemm_with_config(kw_queue qh, int cfg, size_t m, size_t n, size_t k, double alpha, const double* A,
                               size_t lda, const double* B, size_t ldb, double beta, double* C, size_t ldc)
{
    KW_CHECK_QUEUE(qh);
    KW_ENQUEUE_LOCK(qh);
    auto* q = reinterpret_cast<kw::Queue*>(qh);
    if (cfg < 0 || cfg >= kNumCfgs)
        return kw::usage("dgemm config index out of range");
    kw_status st = validate_gemm(m, n, k, A, lda, B, ldb, C, ldc);
    if (st != KW_OK || m == 0 || n == 0)
        return st;
    kw::DeviceGuard g(q->device);
    st = device_operands(q, "dgemm_with_config", k, A, B, C);
    if (st != KW_OK)
        return st;
    st = kCfgs[cfg].launch(q->stream, make_params(m, n, k, alpha, A, lda, B, ldb, beta, C, ldc));
    if (st != KW_OK)
        return kw::task_fail(q, kw::last_error());
    return kw::after_enqueue(q, "dgemm");
}

kw_status kw_dgemm_naive(kw_queue qh, const kw_workdiv* wd, size_t m, size_t n, size_t k, double alpha,
                         const double* A, size_t lda, const double* B, size_t ldb, double beta, double* C, size_t ldc)
{
    KW_CHECK_QUEUE(qh);
    KW_ENQUEUE_LOCK(qh);
    KW_NVTX("kw dgemm (naive)");
    auto* q = reinterpret_cast<kw::Queue*>(qh);
    kw_status st = validate_gemm(m, n, k, A, lda, B, ldb, C, ldc);
    if (st != KW_OK)
        return st;
    kw_workdiv def = {};
    if (wd == nullptr) {
        // GPU thread-level shape of gemmNaiveWorkDiv: (1, 1) elements, 8 x 32 threads.
        def.dim = 2;
        for (int i = 0; i < 3; ++i)
            def.blocks[i] = def.threads[i] = def.elems[i] = 1;
        def.threads[0] = 8;
        def.threads[1] = 32;
        def.blocks[0] = kw::ceil_div(m == 0 ? 1 : m, 8);
        def.blocks[1] = kw::ceil_div(n == 0 ? 1 : n, 32);
        wd = &def;
    }
    if (wd->dim != 2)
        return kw::usage("dgemm_naive: the naive kernel runs on a 2-D (rows, cols) work division");
    for (int i = 0; i < 2; ++i)
        if (wd->blocks[i] == 0 || wd->threads[i] == 0 || wd->elems[i] == 0)
            return kw::usage("WorkDiv: every level extent is at least 1");
    if (wd->threads[0] * wd->threads[1] > 1024 || wd->threads[1] > 1024 || wd->threads[0] > 1024)
        return kw::usage("dgemm_naive: threadsPerBlock exceeds the sm_100a block limit of 1024");
    if (wd->blocks[0] > 65535 || wd->blocks[1] > static_cast<size_t>(INT_MAX))
        return kw::usage("dgemm_naive: blocksPerGrid exceeds the grid limits");
    if (wd->elems[0] > INT_MAX || wd->elems[1] > INT_MAX)
        return kw::usage("dgemm_naive: elementsPerThread too large");
    if (m == 0 || n == 0)
        return KW_OK;
    kw::DeviceGuard g(q->device);
    st = device_operands(q, "dgemm_naive", k, A, B, C);
    if (st != KW_OK)
        return st;
    dim3 grid(static_cast<unsigned>(wd->blocks[1]), static_cast<unsigned>(wd->blocks[0]));
    dim3 block(static_cast<unsigned>(wd->threads[1]), static_cast<unsigned>(wd->threads[0]));
    int er = static_cast<int>(wd->elems[0]), ec = static_cast<int>(wd->elems[1]);
    // A reference thread's er x ec chunk becomes er x ec CUDA threads when the block's outputs fit
    // one CUDA block: the same block tile, one output per CUDA thread (the kernel hands a block's
    // outputs to its threads in column order, so this only changes how many threads share them).
    const size_t tile_rows = wd->threads[0] * wd->elems[0], tile_cols = wd->threads[1] * wd->elems[1];
    if (tile_rows * tile_cols <= 1024) {
        block = dim3(static_cast<unsigned>(tile_cols), static_cast<unsigned>(tile_rows));
        er = ec = 1;
    }
    dgemm_naive_kernel<<<grid, block, 0, q->stream>>>(make_params(m, n, k, alpha, A, lda, B, ldb, beta, C, ldc), er,
                                                       ec);
    kw::g_launches.fetch_add(1, std::memory_order_relaxed);
    return kw::after_enqueue(q, "dgemm_naive");
}

} // extern "C"
