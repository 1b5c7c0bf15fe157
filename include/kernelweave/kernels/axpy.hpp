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

/// Device-usable form of AxpyArgsT: raw element pointers, captured by value by a functor
/// (AxpyArgsT holds host-side Buffer objects, which device code cannot dereference).
template <class T>
struct AxpyArgsView {
    std::size_t n = 0;
    T alpha = T(0);
    const T* x = nullptr;
    T* y = nullptr;
};

template <class T>
inline AxpyArgsView<T> toView(const AxpyArgsT<T>& a)
{
    if (!a.x || !a.y)
        throw UsageError("AxpyArgs: null buffer");
    return AxpyArgsView<T>{a.n, a.alpha, a.x->template rowData<T>(0), a.y->template rowData<T>(0)};
}

namespace detail_ops {
/// fl(fl(a * x) + y): the product and the sum rounded separately, never contracted to an FMA
/// (the reference's SSE mulpd/addpd).
template <class T>
KW_HD inline T mulThenAdd(T a, T x, T y)
{
#if defined(__CUDA_ARCH__)
    if constexpr (sizeof(T) == 4)
        return __fadd_rn(__fmul_rn(a, x), y);
    else
        return __dadd_rn(__dmul_rn(a, x), y);
#else
    volatile T p = a * x; // volatile: the host compiler may not fuse it into an FMA either
    return p + y;
#endif
}
} // namespace detail_ops

/// Element-extended AXPY functor (axpy.hpp:20-26, axpy.cpp:10-23).
///
/// executeTask / createExec never call operator(): they dispatch to the tuned sm_100a kernel
/// (kw_axpy_f32/_f64; each block covers the reference block's elements, the element level as
/// 128-bit vectors). operator() is the reference's per-invocation body, for code that invokes
/// or composes the functor itself:
///   * device form (view args): grid thread g updates [g*V, g*V + min(V, n - g*V)) — call it
///     from a KW_DEVICE_FUNCTOR functor; bit-exact against axpyReference;
///   * reference signature (const AccContext&, const AxpyArgs&): the same body on HOST buffers,
///     run where the call is made (one invocation, as the reference's runGrid calls it).
struct AxpyKernel {
    template <class T>
    KW_HD void operator()(const AccContext& acc, const AxpyArgsView<T>& a) const
    {
        // the paper's spelling: idx::getIdx<Grid, Threads>(acc)[0u]
        const std::size_t gridThreadIdx = idx::getIdx<Grid, Threads>(acc)[0u];
        const std::size_t threadElemExtent = workdiv::getWorkDiv<Thread, Elems>(acc)[0u];
        const std::size_t first = gridThreadIdx * threadElemExtent;
        if (first >= a.n)
            return;
        const std::size_t elems = threadElemExtent < a.n - first ? threadElemExtent : a.n - first;
        for (std::size_t i = first; i < first + elems; ++i)
            a.y[i] = detail_ops::mulThenAdd(a.alpha, a.x[i], a.y[i]);
    }
    template <class T>
    void operator()(const AccContext& acc, const AxpyArgsT<T>& a) const
    {
        const AxpyArgsView<T> v = toView(a);
        if (!a.x->device().isHost() || !a.y->device().isHost())
            throw UsageError("AxpyKernel: a direct call runs one invocation where it is made and needs host "
                             "buffers; GPU buffers go through executeTask / createExec (or the view form inside a "
                             "device functor)");
        (*this)(acc, v);
    }
};

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
