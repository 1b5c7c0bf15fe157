/* kernelweave B200 drop-in — AXPY (reference: core/include/kernelweave/kernels/axpy.hpp,
 * core/src/kernels/axpy.cpp). Y <- alpha * X + Y, bit-exact against axpyReference: products
 * and sums are rounded separately (no FMA), on the sm_100a kernel behind kw_axpy_f32/_f64. */
#pragma once

#include "kernelweave/acc.hpp"
#include "kernelweave/buffer.hpp"
#include "kernelweave/exec.hpp"

namespace kernelweave::kernels {

/// AxpyArgs (axpy.hpp:13-18) generalised over the element type; AxpyArgs keeps the reference's
/// fp64 layout, AxpyArgsF32 is the fp32 path BASELINE.json measures.
template <class T>
struct AxpyArgsT {
    std::size_t n = 0;
    T alpha = T(0);
    const Buffer* x = nullptr;
    Buffer* y = nullptr;
};
using AxpyArgs = AxpyArgsT<double>;
using AxpyArgsF32 = AxpyArgsT<float>;

/// Element-extended AXPY functor (axpy.hpp:20-26). On GpuCudaRt each block covers the same
/// elements as the reference block; the element level becomes 128-bit vectors per thread.
struct AxpyKernel {};

/// axpy.cpp:25-30.
inline WorkDiv axpyWorkDiv(BackendKind backend, std::size_t n, std::size_t threadsPerBlock,
                           std::size_t elementsPerThread)
{
    return divideForBackend(IndexVec(n), backend, IndexVec(threadsPerBlock), IndexVec(elementsPerThread));
}

} // namespace kernelweave::kernels

namespace kernelweave::detail {

template <class T>
struct Launcher<kernels::AxpyKernel, kernels::AxpyArgsT<T>> {
    static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>, "AXPY is fp32 or fp64");
    static void validate(const WorkDiv& wd, const kernels::AxpyArgsT<T>& a)
    {
        if (!a.x || !a.y)
            throw UsageError("AxpyArgs: null buffer");
        if (a.x->elemSize() != sizeof(T) || a.y->elemSize() != sizeof(T))
            throw UsageError("Buffer: typed access with mismatching element size");
        if (a.n > a.x->extent().product() || a.n > a.y->extent().product())
            throw UsageError("axpy: n exceeds a buffer extent");
        if (wd.dim() != 1)
            throw UsageError("axpy: the AXPY kernel runs on a 1-D work division");
    }
    static kw_status launch(kw_queue q, const WorkDiv& wd, const kernels::AxpyKernel&, const kernels::AxpyArgsT<T>& a)
    {
        const kw_workdiv w = wd.toC();
        if constexpr (std::is_same_v<T, float>)
            return kw_axpy_f32(q, &w, a.n, a.alpha, a.x->template rowData<float>(0), a.y->template rowData<float>(0));
        else
            return kw_axpy_f64(q, &w, a.n, a.alpha, a.x->template rowData<double>(0),
                               a.y->template rowData<double>(0));
    }
    static Device device(const kernels::AxpyArgsT<T>& a) { return a.y->device(); }
};

} // namespace kernelweave::detail
