/* kernelweave B200 drop-in — work division (reference: core/include/kernelweave/work_div.hpp,
 * core/src/work_div.cpp:53-119). */
#pragma once

#include "kernelweave/backend.hpp"
#include "kernelweave/index_vec.hpp"

#include <string>

namespace kernelweave {

enum class Level { Grid, Block, Thread };
enum class Unit { Blocks, Threads, Elems };

inline std::string_view name(Level l) { return l == Level::Grid ? "Grid" : l == Level::Block ? "Block" : "Thread"; }
inline std::string_view name(Unit u) { return u == Unit::Blocks ? "Blocks" : u == Unit::Threads ? "Threads" : "Elems"; }

class WorkDiv {
public:
    WorkDiv(IndexVec blocksPerGrid, IndexVec threadsPerBlock, IndexVec elementsPerThread)
        : m_b(blocksPerGrid), m_t(threadsPerBlock), m_e(elementsPerThread)
    {
        detail::requireSameDim(m_b, m_t, "WorkDiv");
        detail::requireSameDim(m_b, m_e, "WorkDiv");
        requirePositive(m_b, "blocksPerGrid");
        requirePositive(m_t, "threadsPerBlock");
        requirePositive(m_e, "elementsPerThread");
    }

    const IndexVec& blocksPerGrid() const noexcept { return m_b; }
    const IndexVec& threadsPerBlock() const noexcept { return m_t; }
    const IndexVec& elementsPerThread() const noexcept { return m_e; }
    std::size_t dim() const noexcept { return m_b.dim(); }

    friend bool operator==(const WorkDiv& a, const WorkDiv& b) noexcept
    {
        return a.m_b == b.m_b && a.m_t == b.m_t && a.m_e == b.m_e;
    }

    /// The C-ABI view.
    kw_workdiv toC() const noexcept
    {
        kw_workdiv w{};
        w.dim = static_cast<uint32_t>(dim());
        const auto b = m_b.padded(), t = m_t.padded(), e = m_e.padded();
        for (int k = 0; k < 3; ++k) {
            w.blocks[k] = b[k];
            w.threads[k] = t[k];
            w.elems[k] = e[k];
        }
        return w;
    }

    static WorkDiv fromC(const kw_workdiv& w)
    {
        auto iv = [&](const size_t* v) {
            return w.dim == 1 ? IndexVec(v[0]) : w.dim == 2 ? IndexVec(v[0], v[1]) : IndexVec(v[0], v[1], v[2]);
        };
        return WorkDiv(iv(w.blocks), iv(w.threads), iv(w.elems));
    }

private:
    static void requirePositive(const IndexVec& v, const char* what)
    {
        for (std::size_t k = 0; k < v.dim(); ++k)
            if (v[k] == 0)
                throw UsageError(std::string("WorkDiv: ") + what +
                                 " has a zero component; every level extent is at least 1");
    }
    IndexVec m_b, m_t, m_e;
};

/// work_div.cpp:65-94.
inline IndexVec totalExtent(const WorkDiv& wd, Level origin, Unit unit)
{
    if (origin == Level::Grid && unit == Unit::Blocks)
        return wd.blocksPerGrid();
    if (origin == Level::Grid && unit == Unit::Threads)
        return wd.blocksPerGrid() * wd.threadsPerBlock();
    if (origin == Level::Grid && unit == Unit::Elems)
        return wd.blocksPerGrid() * wd.threadsPerBlock() * wd.elementsPerThread();
    if (origin == Level::Block && unit == Unit::Threads)
        return wd.threadsPerBlock();
    if (origin == Level::Block && unit == Unit::Elems)
        return wd.threadsPerBlock() * wd.elementsPerThread();
    if (origin == Level::Thread && unit == Unit::Elems)
        return wd.elementsPerThread();
    throw UsageError("totalExtent: unsupported (origin, unit) pair (" + std::string(name(origin)) + ", " +
                     std::string(name(unit)) + ")");
}

/// work_div.cpp:96-119. GpuCudaRt takes the thread-level shape ceil(N/(B*V)) x B x V.
inline WorkDiv divideForBackend(const IndexVec& problem, BackendKind backend, const IndexVec& threadsHint,
                                const IndexVec& elemsHint)
{
    detail::requireSameDim(problem, threadsHint, "divideForBackend");
    detail::requireSameDim(problem, elemsHint, "divideForBackend");
    for (const auto* v : {&problem, &threadsHint, &elemsHint})
        for (std::size_t k = 0; k < v->dim(); ++k)
            if ((*v)[k] == 0)
                throw UsageError("WorkDiv: a zero component; every level extent is at least 1");
    const IndexVec ones = IndexVec::filled(problem.dim(), 1);
    switch (backend) {
    case BackendKind::Serial:
    case BackendKind::BlocksParallel:
        return WorkDiv(ceilDivide(problem, elemsHint), ones, elemsHint);
    case BackendKind::ThreadsParallel:
    case BackendKind::GpuCudaRt:
        return WorkDiv(ceilDivide(problem, threadsHint * elemsHint), threadsHint, elemsHint);
    }
    throw UsageError("divideForBackend: unknown BackendKind value");
}

} // namespace kernelweave
