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

struct GemmNaiveKernel {};
struct GemmTiledKernel {};

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
