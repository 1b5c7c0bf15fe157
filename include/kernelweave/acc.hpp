/* kernelweave B200 drop-in — kernel-side accelerator API (reference:
 * core/include/kernelweave/acc.hpp, core/src/accel.cpp:269-321).
 *
 * AccContext is the per-(block, thread) handle a functor receives. In this build it is a small
 * trivially-copyable value usable in device code (kernelweave/cuda_exec.cuh constructs it from
 * the CUDA built-ins); on the host it can be built explicitly to evaluate the index algebra.
 * Both spellings of the index queries are provided and must agree (test_accel.cpp:61-86):
 *   getIdx(acc, Level::Grid, Unit::Threads)          (kernelweave's enum form)
 *   idx::getIdx<Grid, Threads>(acc)                  (the paper's template-tag form; invalid
 *                                                     pairs fail at compile time) */
#pragma once

#include "kernelweave/work_div.hpp"

#include <cstdint>
#include <string>

namespace kernelweave {

class AccContext {
public:
    AccContext(const WorkDiv& wd, const IndexVec& gridBlockIdx, const IndexVec& blockThreadIdx)
        : m_wd(wd.toC()), m_block(gridBlockIdx), m_thread(blockThreadIdx)
    {
        detail::requireSameDim(gridBlockIdx, blockThreadIdx, "AccContext");
        if (gridBlockIdx.dim() != wd.dim())
            throw UsageError("AccContext: index and work-division dimensionalities differ");
    }
    KW_HD AccContext(const kw_workdiv& wd, const IndexVec& gridBlockIdx, const IndexVec& blockThreadIdx,
                     std::byte* shared = nullptr, std::size_t sharedBytes = 0,
                     std::uint32_t* failSlot = nullptr) noexcept
        : m_wd(wd), m_block(gridBlockIdx), m_thread(blockThreadIdx), m_shared(shared), m_sharedBytes(sharedBytes),
          m_fail(failSlot)
    {
    }
    AccContext(const AccContext&) = default;

    KW_HD const kw_workdiv& workDiv() const noexcept { return m_wd; }
    KW_HD const IndexVec& gridBlockIdx() const noexcept { return m_block; }
    KW_HD const IndexVec& blockThreadIdx() const noexcept { return m_thread; }

    // Block shared-memory arena (device launches, kernelweave/cuda_exec.cuh): allocation calls
    // are matched across a block's threads by sequence, exactly like SharedArena
    // (accel.cpp:24-61) — every thread issues the same sequence and so computes the same offsets.
    KW_HD std::byte* sharedBase() const noexcept { return m_shared; }
    KW_HD std::size_t sharedBytes() const noexcept { return m_sharedBytes; }
    KW_HD std::size_t& sharedCursor() const noexcept { return m_cursor; }
    // Device launches: the task's failure slot (kw_queue_fail_slot), set by failTask().
    KW_HD std::uint32_t* failSlot() const noexcept { return m_fail; }

private:
    kw_workdiv m_wd;
    IndexVec m_block;
    IndexVec m_thread;
    std::byte* m_shared = nullptr;
    std::size_t m_sharedBytes = 0;
    std::uint32_t* m_fail = nullptr;
    mutable std::size_t m_cursor = 0;
};

namespace detail {
KW_HD inline IndexVec make(std::size_t dim, const std::size_t* v) noexcept
{
    return dim == 1 ? IndexVec(v[0]) : dim == 2 ? IndexVec(v[0], v[1]) : IndexVec(v[0], v[1], v[2]);
}
/// a * b + c component-wise (b a size_t[3] of the work division); array-free for device code.
KW_HD inline IndexVec mulAdd(const IndexVec& a, const std::size_t* b, const IndexVec& c) noexcept
{
    const std::size_t d = a.dim();
    const std::size_t x0 = a.get(0) * b[0] + c.get(0);
    if (d == 1)
        return IndexVec(x0);
    const std::size_t x1 = a.get(1) * b[1] + c.get(1);
    if (d == 2)
        return IndexVec(x0, x1);
    return IndexVec(x0, x1, a.get(2) * b[2] + c.get(2));
}
/// One (origin, unit) extent component of a work division (totalExtent, work_div.cpp:65-94).
KW_HD inline std::size_t extentComponent(const kw_workdiv& w, std::size_t k, Level origin, Unit unit) noexcept
{
    std::size_t v = 1;
    if (origin == Level::Grid)
        v *= w.blocks[k];
    if (origin != Level::Thread && unit != Unit::Blocks)
        v *= w.threads[k];
    if (unit == Unit::Elems)
        v *= w.elems[k];
    return v;
}
} // namespace detail

/// accel.cpp:269-279: (Grid, Blocks), (Grid, Threads) = block * threadsPerBlock + thread,
/// (Block, Threads); any other pair is a usage error (device code: a trap).
KW_HD inline IndexVec getIdx(const AccContext& acc, Level origin, Unit unit)
{
    if (origin == Level::Grid && unit == Unit::Blocks)
        return acc.gridBlockIdx();
    if (origin == Level::Grid && unit == Unit::Threads)
        return detail::mulAdd(acc.gridBlockIdx(), acc.workDiv().threads, acc.blockThreadIdx());
    if (origin == Level::Block && unit == Unit::Threads)
        return acc.blockThreadIdx();
#if defined(__CUDA_ARCH__)
    __trap();
    return acc.gridBlockIdx();
#else
    throw UsageError("getIdx: unsupported (origin, unit) pair (" + std::string(name(origin)) + ", " +
                     std::string(name(unit)) + ")");
#endif
}

/// accel.cpp:281-284 → totalExtent (work_div.cpp:65-94).
KW_HD inline IndexVec getWorkDiv(const AccContext& acc, Level origin, Unit unit)
{
    const kw_workdiv& w = acc.workDiv();
    const bool ok = (origin == Level::Grid) || (origin == Level::Block && unit != Unit::Blocks) ||
                    (origin == Level::Thread && unit == Unit::Elems);
    if (!ok) {
#if defined(__CUDA_ARCH__)
        __trap();
#else
        throw UsageError("totalExtent: unsupported (origin, unit) pair (" + std::string(name(origin)) + ", " +
                         std::string(name(unit)) + ")");
#endif
    }
    const std::size_t e0 = detail::extentComponent(w, 0, origin, unit);
    if (w.dim == 1)
        return IndexVec(e0);
    const std::size_t e1 = detail::extentComponent(w, 1, origin, unit);
    if (w.dim == 2)
        return IndexVec(e0, e1);
    return IndexVec(e0, e1, detail::extentComponent(w, 2, origin, unit));
}

// ---- the paper's template-tag spelling --------------------------------
struct Grid {};
struct Block {};
struct Thread {};
struct Blocks {};
struct Threads {};
struct Elems {};

namespace idx {
template <class Origin, class UnitT>
KW_HD inline IndexVec getIdx(const AccContext& acc) noexcept
{
    if constexpr (std::is_same_v<Origin, Grid> && std::is_same_v<UnitT, Blocks>)
        return acc.gridBlockIdx();
    else if constexpr (std::is_same_v<Origin, Grid> && std::is_same_v<UnitT, Threads>)
        return detail::mulAdd(acc.gridBlockIdx(), acc.workDiv().threads, acc.blockThreadIdx());
    else if constexpr (std::is_same_v<Origin, Block> && std::is_same_v<UnitT, Threads>)
        return acc.blockThreadIdx();
    else
        static_assert(sizeof(Origin) == 0, "getIdx: unsupported (origin, unit) pair");
}
} // namespace idx

namespace workdiv {
template <class Origin, class UnitT>
KW_HD inline IndexVec getWorkDiv(const AccContext& acc) noexcept
{
    constexpr bool valid =
        std::is_same_v<Origin, Grid> || (std::is_same_v<Origin, Block> && !std::is_same_v<UnitT, Blocks>) ||
        (std::is_same_v<Origin, Thread> && std::is_same_v<UnitT, Elems>);
    static_assert(valid, "getWorkDiv: unsupported (origin, unit) pair");
    constexpr Level o = std::is_same_v<Origin, Grid> ? Level::Grid
                        : std::is_same_v<Origin, Block> ? Level::Block
                                                        : Level::Thread;
    constexpr Unit u = std::is_same_v<UnitT, Blocks> ? Unit::Blocks
                       : std::is_same_v<UnitT, Threads> ? Unit::Threads
                                                        : Unit::Elems;
    const kw_workdiv& w = acc.workDiv();
    const std::size_t e0 = detail::extentComponent(w, 0, o, u);
    if (w.dim == 1)
        return IndexVec(e0);
    const std::size_t e1 = detail::extentComponent(w, 1, o, u);
    if (w.dim == 2)
        return IndexVec(e0, e1);
    return IndexVec(e0, e1, detail::extentComponent(w, 2, o, u));
}
} // namespace workdiv

#if !defined(__CUDACC__)
// Kernel-side services for host-compiled translation units (acc.hpp:84-106 declarations). This
// build has no CPU back-end: a functor that uses them runs on the GPU only, compiled by nvcc
// against kernelweave/cuda_exec.cuh (which defines the device versions). A host-compiled
// functor still compiles; calling these on the host is a usage error.
[[noreturn]] inline void hostKernelServiceUnavailable(const char* what)
{
    throw UsageError(std::string(what) +
                     ": kernel-side service of a device functor — compile the functor with nvcc against "
                     "kernelweave/cuda_exec.cuh (there is no CPU back-end in the B200 build)");
}
inline void* allocSharedMem(const AccContext&, std::size_t, std::size_t) { hostKernelServiceUnavailable("allocSharedMem"); }
template <class T>
T* allocSharedMem(const AccContext& acc, std::size_t count)
{
    return static_cast<T*>(allocSharedMem(acc, count, sizeof(T)));
}
inline void syncBlockThreads(const AccContext&) { hostKernelServiceUnavailable("syncBlockThreads"); }
inline double atomicAdd(const AccContext&, double&, double) { hostKernelServiceUnavailable("atomicAdd"); }
inline std::int64_t atomicAdd(const AccContext&, std::int64_t&, std::int64_t)
{
    hostKernelServiceUnavailable("atomicAdd");
}
inline std::uint64_t atomicAdd(const AccContext&, std::uint64_t&, std::uint64_t)
{
    hostKernelServiceUnavailable("atomicAdd");
}
#endif

} // namespace kernelweave
