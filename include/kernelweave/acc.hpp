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
                     std::byte* shared = nullptr, std::size_t sharedBytes = 0) noexcept
        : m_wd(wd), m_block(gridBlockIdx), m_thread(blockThreadIdx), m_shared(shared), m_sharedBytes(sharedBytes)
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

private:
    kw_workdiv m_wd;
    IndexVec m_block;
    IndexVec m_thread;
    std::byte* m_shared = nullptr;
    std::size_t m_sharedBytes = 0;
    mutable std::size_t m_cursor = 0;
};

namespace detail {
KW_HD inline IndexVec make(std::size_t dim, const std::size_t* v) noexcept
{
    return dim == 1 ? IndexVec(v[0]) : dim == 2 ? IndexVec(v[0], v[1]) : IndexVec(v[0], v[1], v[2]);
}
KW_HD inline IndexVec mulAdd(const IndexVec& a, const std::size_t* b, const IndexVec& c) noexcept
{
    std::size_t r[3] = {0, 0, 0};
    for (std::size_t k = 0; k < a.dim(); ++k)
        r[k] = a.get(k) * b[k] + c.get(k);
    return make(a.dim(), r);
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
    std::size_t r[3] = {1, 1, 1};
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
    for (uint32_t k = 0; k < w.dim; ++k) {
        std::size_t v = 1;
        if (origin == Level::Grid)
            v *= w.blocks[k];
        if (origin != Level::Thread && unit != Unit::Blocks)
            v *= w.threads[k];
        if (unit == Unit::Elems)
            v *= w.elems[k];
        r[k] = v;
    }
    return detail::make(w.dim, r);
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
    const kw_workdiv& w = acc.workDiv();
    std::size_t r[3];
    for (uint32_t k = 0; k < 3; ++k) {
        if constexpr (std::is_same_v<Origin, Grid> && std::is_same_v<UnitT, Blocks>)
            r[k] = w.blocks[k];
        else if constexpr (std::is_same_v<Origin, Grid> && std::is_same_v<UnitT, Threads>)
            r[k] = w.blocks[k] * w.threads[k];
        else if constexpr (std::is_same_v<Origin, Grid> && std::is_same_v<UnitT, Elems>)
            r[k] = w.blocks[k] * w.threads[k] * w.elems[k];
        else if constexpr (std::is_same_v<Origin, Block> && std::is_same_v<UnitT, Threads>)
            r[k] = w.threads[k];
        else if constexpr (std::is_same_v<Origin, Block> && std::is_same_v<UnitT, Elems>)
            r[k] = w.threads[k] * w.elems[k];
        else if constexpr (std::is_same_v<Origin, Thread> && std::is_same_v<UnitT, Elems>)
            r[k] = w.elems[k];
        else
            static_assert(sizeof(Origin) == 0, "getWorkDiv: unsupported (origin, unit) pair");
    }
    return detail::make(w.dim, r);
}
} // namespace workdiv

} // namespace kernelweave
