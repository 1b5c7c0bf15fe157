/* kernelweave B200 drop-in — DGEMM (reference: core/include/kernelweave/kernels/gemm.hpp,
 * core/src/kernels/gemm.cpp). C <- alpha * A * B + beta * C on pitched row-major fp64 buffers.
 *   GemmTiledKernel: FP64 DMMA tensor-core kernel (TMA + mbarrier pipeline), within
 *                    |dC| <= (K+4) 2^-53 |C_ref| of gemmReference;
 *   GemmNaiveKernel: one ascending-p dot product per output with separately rounded products
 *                    and sums — bitwise identical to gemmReference. */
#pragma once

#include "kernelweave/acc.hpp"
#include "kernelweave/buffer.hpp"
#include "kernelweave/exec.hpp"

#include <string>

namespace kernelweave::kernels {

/// gemm.hpp:16-26. On GpuCudaRt `tile` is the DMMA block tile edge (64 or 128).
struct GemmArgs {
    std::size_t m = 0;
    std::size_t n = 0;
    std::size_t k = 0;
    double alpha = 0.0;
    double beta = 0.0;
    const Buffer* a = nullptr;
    const Buffer* b = nullptr;
    Buffer* c = nullptr;
    std::size_t tile = 128;
    /// GemmTiledKernel only: bit-exact mode — separately rounded products and sums in
    /// ascending k, bitwise equal to gemmReference (FP64-pipe bound, about half the DMMA rate).
    bool bitwise = false;
};

/// Device-usable form of GemmArgs (element pointers and leading dimensions, by value).
struct GemmArgsView {
    std::size_t m = 0, n = 0, k = 0;
    double alpha = 0.0, beta = 0.0;
    const double* a = nullptr;
    std::size_t lda = 0;
    const double* b = nullptr;
    std::size_t ldb = 0;
    double* c = nullptr;
    std::size_t ldc = 0;
    std::size_t tile = 16;
};

inline GemmArgsView toView(const GemmArgs& g)
{
    if (!g.a || !g.b || !g.c)
        throw UsageError("GemmArgs: null buffer");
    return GemmArgsView{g.m, g.n, g.k, g.alpha, g.beta, g.a->rowData<double>(0), g.a->leadingDim<double>(),
                        g.b->rowData<double>(0), g.b->leadingDim<double>(), g.c->rowData<double>(0),
                        g.c->leadingDim<double>(), g.tile};
}

namespace detail_ops {
KW_HD inline double mul(double a, double b)
{
#if defined(__CUDA_ARCH__)
    return __dmul_rn(a, b);
#else
    volatile double p = a * b;
    return p;
#endif
}
KW_HD inline double add(double a, double b)
{
#if defined(__CUDA_ARCH__)
    return __dadd_rn(a, b);
#else
    return a + b;
#endif
}
inline void requireHostOperands(const GemmArgs& g, const char* who)
{
    if (!g.a->device().isHost() || !g.b->device().isHost() || !g.c->device().isHost())
        throw UsageError(std::string(who) + ": a direct call runs one invocation where it is made and needs host "
                                            "buffers; GPU buffers go through executeTask / createExec (or the view "
                                            "form inside a device functor)");
}
} // namespace detail_ops

/// Naive DGEMM functor (gemm.hpp:28-34, gemm.cpp:11-38). executeTask dispatches to the tuned
/// kernel (kw_dgemm_naive); operator() is the reference's per-invocation body — view form for
/// device functors, reference signature on host buffers — bitwise equal to gemmReference:
/// ascending-p sum of separately rounded products from +0.0, then fl(fl(a*acc) + fl(b*c)).
struct GemmNaiveKernel {
    KW_HD void operator()(const AccContext& acc, const GemmArgsView& g) const
    {
        const IndexVec gt = idx::getIdx<Grid, Threads>(acc);
        const IndexVec ept = workdiv::getWorkDiv<Thread, Elems>(acc);
        const std::size_t rowFirst = gt.get(0) * ept.get(0);
        const std::size_t colFirst = gt.get(1) * ept.get(1);
        if (rowFirst >= g.m || colFirst >= g.n)
            return;
        const std::size_t rowEnd = rowFirst + ept.get(0) < g.m ? rowFirst + ept.get(0) : g.m;
        const std::size_t colEnd = colFirst + ept.get(1) < g.n ? colFirst + ept.get(1) : g.n;
        for (std::size_t r = rowFirst; r < rowEnd; ++r)
            for (std::size_t col = colFirst; col < colEnd; ++col) {
                double acc0 = 0.0;
                for (std::size_t p = 0; p < g.k; ++p)
                    acc0 = detail_ops::add(acc0, detail_ops::mul(g.a[r * g.lda + p], g.b[p * g.ldb + col]));
                double* cell = g.c + r * g.ldc + col;
                *cell = detail_ops::add(detail_ops::mul(g.alpha, acc0), detail_ops::mul(g.beta, *cell));
            }
    }
    void operator()(const AccContext& acc, const GemmArgs& g) const
    {
        const GemmArgsView v = toView(g);
        detail_ops::requireHostOperands(g, "GemmNaiveKernel");
        (*this)(acc, v);
    }
};

/// Tiled DGEMM functor (gemm.hpp:36-49, gemm.cpp:40-118). executeTask dispatches to the FP64
/// DMMA kernel (or, with GemmArgs::bitwise, the bit-exact tiled kernel). operator() is the
/// reference's block-cooperative body for device functors: A and B tiles staged in
/// allocSharedMem regions with zero padding by the threads owning the first column chunk, a
/// barrier, ascending-p partial sums, a barrier per k-step, then the alpha/beta epilogue — bitwise
/// equal to gemmReference. The per-thread partials (a std::vector in the reference) live in a
/// third shared region, so the functor needs 3 * tile^2 doubles of block shared memory.
/// There is no host form: the body is block-cooperative, and this build has no CPU back-end
/// (the reference signature compiles and reports a UsageError).
struct GemmTiledKernel {
    template <class Acc>
    KW_HD void operator()(const Acc& acc, const GemmArgsView& g) const
    {
#if defined(__CUDA_ARCH__)
        const std::size_t tile = g.tile;
        // (untemplated spelling: the services are found by ADL once Acc is known)
        double* tileA = static_cast<double*>(allocSharedMem(acc, tile * tile, sizeof(double)));
        double* tileB = static_cast<double*>(allocSharedMem(acc, tile * tile, sizeof(double)));
        double* part = static_cast<double*>(allocSharedMem(acc, tile * tile, sizeof(double))); // zeroed: sums start at +0.0
        const IndexVec blk = idx::getIdx<Grid, Blocks>(acc);
        const IndexVec thr = idx::getIdx<Block, Threads>(acc);
        const IndexVec ept = workdiv::getWorkDiv<Thread, Elems>(acc);
        const std::size_t rowBase = blk.get(0) * tile, colBase = blk.get(1) * tile;
        auto clamp = [tile](std::size_t v) { return v < tile ? v : tile; };
        const std::size_t tr0 = clamp(thr.get(0) * ept.get(0)), tc0 = clamp(thr.get(1) * ept.get(1));
        const std::size_t trEnd = clamp(tr0 + ept.get(0)), tcEnd = clamp(tc0 + ept.get(1));
        const std::size_t kSteps = (g.k + tile - 1) / tile;
        for (std::size_t step = 0; step < kSteps; ++step) {
            const std::size_t kBase = step * tile;
            if (tc0 == 0) {
                for (std::size_t sr = tr0; sr < trEnd; ++sr) {
                    const std::size_t aRow = rowBase + sr, bRow = kBase + sr;
                    for (std::size_t j = 0; j < tile; ++j) {
                        const std::size_t aCol = kBase + j, bCol = colBase + j;
                        tileA[sr * tile + j] = (aRow < g.m && aCol < g.k) ? g.a[aRow * g.lda + aCol] : 0.0;
                        tileB[sr * tile + j] = (bRow < g.k && bCol < g.n) ? g.b[bRow * g.ldb + bCol] : 0.0;
                    }
                }
            }
            syncBlockThreads(acc);
            for (std::size_t r = tr0; r < trEnd; ++r)
                for (std::size_t col = tc0; col < tcEnd; ++col) {
                    double sum = part[r * tile + col];
                    for (std::size_t p = 0; p < tile; ++p)
                        sum = detail_ops::add(sum, detail_ops::mul(tileA[r * tile + p], tileB[p * tile + col]));
                    part[r * tile + col] = sum;
                }
            syncBlockThreads(acc);
        }
        for (std::size_t r = tr0; r < trEnd; ++r) {
            const std::size_t outRow = rowBase + r;
            if (outRow >= g.m)
                break;
            for (std::size_t col = tc0; col < tcEnd; ++col) {
                const std::size_t outCol = colBase + col;
                if (outCol >= g.n)
                    break;
                double* cell = g.c + outRow * g.ldc + outCol;
                *cell = detail_ops::add(detail_ops::mul(g.alpha, part[r * tile + col]), detail_ops::mul(g.beta, *cell));
            }
        }
#else
        (void)acc;
        (void)g;
        throw UsageError("GemmTiledKernel: the tiled body is block-cooperative (allocSharedMem, "
                         "syncBlockThreads) and runs in device functors only; use executeTask / createExec");
#endif
    }
    template <class Acc>
    void operator()(const Acc& acc, const GemmArgs& g) const
    {
        (*this)(acc, toView(g));
    }
};

/// gemm.cpp:120-125.
inline WorkDiv gemmNaiveWorkDiv(BackendKind backend, std::size_t m, std::size_t n, std::size_t threadsPerBlock,
                                std::size_t elementsPerThread)
{
    return divideForBackend(IndexVec(m, n), backend, IndexVec(threadsPerBlock, 1), IndexVec(1, elementsPerThread));
}

/// gemm.cpp:127-135; GpuCudaRt: one block per tile x tile output tile of the DMMA kernel.
inline WorkDiv gemmTiledWorkDiv(BackendKind backend, std::size_t m, std::size_t n, std::size_t tile)
{
    if (tile == 0)
        throw UsageError("gemmTiledWorkDiv: tile edge must be positive");
    const IndexVec blocks((m + tile - 1) / tile, (n + tile - 1) / tile);
    if (backend == BackendKind::GpuCudaRt) {
        kw_workdiv w{};
        detail::check(kw_dgemm_default_workdiv(m, n, tile, &w));
        return WorkDiv::fromC(w);
    }
    if (backend == BackendKind::ThreadsParallel)
        return WorkDiv(blocks, IndexVec(tile, 1), IndexVec(1, tile));
    return WorkDiv(blocks, IndexVec(1, 1), IndexVec(tile, tile));
}

} // namespace kernelweave::kernels

namespace kernelweave::detail {

struct GemmLauncherBase {
    static void validate(const WorkDiv& wd, const kernels::GemmArgs& a)
    {
        if (!a.a || !a.b || !a.c)
            throw UsageError("GemmArgs: null buffer");
        for (const Buffer* b : {a.a, a.b, static_cast<const Buffer*>(a.c)})
            if (b->elemSize() != sizeof(double) || b->dim() != 2)
                throw UsageError("Buffer: typed access with mismatching element size");
        if (a.k > 0 && (a.a->extent()[0] < a.m || a.a->extent()[1] < a.k || a.b->extent()[0] < a.k ||
                        a.b->extent()[1] < a.n))
            throw UsageError("gemm: extents exceed a buffer extent");
        if (a.c->extent()[0] < a.m || a.c->extent()[1] < a.n)
            throw UsageError("gemm: extents exceed a buffer extent");
        if (wd.dim() != 2)
            throw UsageError("gemm: the GEMM kernels run on a 2-D (rows, cols) work division");
    }
    static Device device(const kernels::GemmArgs& a) { return a.c->device(); }
};

template <>
struct Launcher<kernels::GemmTiledKernel, kernels::GemmArgs> : GemmLauncherBase {
    static kw_status launch(kw_queue q, const WorkDiv& wd, const kernels::GemmTiledKernel&,
                            const kernels::GemmArgs& a)
    {
        const kw_workdiv w = wd.toC();
        if (a.bitwise)
            return kw_dgemm_bitwise(q, &w, a.m, a.n, a.k, a.alpha, a.a->rowData<double>(0), a.a->leadingDim<double>(),
                                    a.b->rowData<double>(0), a.b->leadingDim<double>(), a.beta,
                                    a.c->rowData<double>(0), a.c->leadingDim<double>());
        return kw_dgemm(q, &w, a.m, a.n, a.k, a.alpha, a.a->rowData<double>(0), a.a->leadingDim<double>(),
                        a.b->rowData<double>(0), a.b->leadingDim<double>(), a.beta, a.c->rowData<double>(0),
                        a.c->leadingDim<double>());
    }
};

template <>
struct Launcher<kernels::GemmNaiveKernel, kernels::GemmArgs> : GemmLauncherBase {
    static kw_status launch(kw_queue q, const WorkDiv& wd, const kernels::GemmNaiveKernel&,
                            const kernels::GemmArgs& a)
    {
        const kw_workdiv w = wd.toC();
        return kw_dgemm_naive(q, &w, a.m, a.n, a.k, a.alpha, a.a->rowData<double>(0), a.a->leadingDim<double>(),
                              a.b->rowData<double>(0), a.b->leadingDim<double>(), a.beta, a.c->rowData<double>(0),
                              a.c->leadingDim<double>());
    }
};

} // namespace kernelweave::detail
