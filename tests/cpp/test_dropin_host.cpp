// Host-only checks of the C++ drop-in (no GPU): index algebra, work division and the
// accelerator index queries, mirroring test_index_vec.cpp, test_work_div.cpp:23-115 and
// test_accel.cpp:61-86 of the reference.
#include <kernelweave/kernelweave.hpp>

#include "check.hpp"

#include <random>

using namespace kernelweave;

TEST_CASE("IndexVec algebra and bounds")
{
    const IndexVec a(2, 3, 4), b(5, 6, 7);
    CHECK((a * b) == IndexVec(10, 18, 28));
    CHECK((a + b) == IndexVec(7, 9, 11));
    CHECK(ceilDivide(IndexVec(100), IndexVec(16)) == IndexVec(7));
    CHECK(a.product() == 24);
    CHECK_THROWS_AS(a[3], UsageError);
    CHECK_THROWS_AS(IndexVec::filled(4, 1), UsageError);
    CHECK_THROWS_AS(ceilDivide(IndexVec(1), IndexVec(0)), UsageError);
    CHECK_THROWS_AS(a * IndexVec(1, 2), UsageError);
    std::mt19937_64 rng(7);
    for (int i = 0; i < 2000; ++i) {
        const IndexVec ext(1 + rng() % 9, 1 + rng() % 9, 1 + rng() % 9);
        const std::size_t lin = rng() % ext.product();
        CHECK(linearize(delinearize(lin, ext), ext) == lin);
    }
    CHECK(delinearize(35, IndexVec(4, 16)) == IndexVec(2, 3));
}

TEST_CASE("totalExtent over all supported pairs (test_work_div.cpp:23-45)")
{
    const WorkDiv wd(IndexVec(3, 5), IndexVec(4, 2), IndexVec(2, 7));
    CHECK(totalExtent(wd, Level::Grid, Unit::Blocks) == IndexVec(3, 5));
    CHECK(totalExtent(wd, Level::Grid, Unit::Threads) == IndexVec(12, 10));
    CHECK(totalExtent(wd, Level::Grid, Unit::Elems) == IndexVec(24, 70));
    CHECK(totalExtent(wd, Level::Block, Unit::Threads) == IndexVec(4, 2));
    CHECK(totalExtent(wd, Level::Block, Unit::Elems) == IndexVec(8, 14));
    CHECK(totalExtent(wd, Level::Thread, Unit::Elems) == IndexVec(2, 7));
    CHECK_THROWS_AS(totalExtent(wd, Level::Thread, Unit::Threads), UsageError);
    CHECK_THROWS_AS(totalExtent(wd, Level::Block, Unit::Blocks), UsageError);
    CHECK_THROWS_AS(WorkDiv(IndexVec(1), IndexVec(0), IndexVec(1)), UsageError);
    CHECK_THROWS_AS(WorkDiv(IndexVec(1), IndexVec(1, 1), IndexVec(1)), UsageError);
}

TEST_CASE("divideForBackend table shapes (test_work_div.cpp:60-115)")
{
    const WorkDiv s = divideForBackend(IndexVec(4096), BackendKind::Serial, IndexVec(16), IndexVec(4));
    CHECK(s.blocksPerGrid() == IndexVec(1024) && s.threadsPerBlock() == IndexVec(1));
    const WorkDiv t = divideForBackend(IndexVec(4096), BackendKind::ThreadsParallel, IndexVec(16), IndexVec(4));
    CHECK(t.blocksPerGrid() == IndexVec(64) && t.threadsPerBlock() == IndexVec(16));
    const WorkDiv g = divideForBackend(IndexVec(4096), BackendKind::GpuCudaRt, IndexVec(256), IndexVec(16));
    CHECK(g.blocksPerGrid() == IndexVec(1) && g.threadsPerBlock() == IndexVec(256));
    CHECK(divideForBackend(IndexVec(100), BackendKind::GpuCudaRt, IndexVec(16), IndexVec(4)).blocksPerGrid() ==
          IndexVec(2));
    std::mt19937_64 rng(86);
    for (int i = 0; i < 1000; ++i) {
        const IndexVec p(1 + rng() % 5000, 1 + rng() % 300);
        const IndexVec th(1 + rng() % 32, 1 + rng() % 32), el(1 + rng() % 8, 1 + rng() % 8);
        const WorkDiv wd = divideForBackend(p, BackendKind::GpuCudaRt, th, el);
        const IndexVec cov = totalExtent(wd, Level::Grid, Unit::Elems);
        for (std::size_t k = 0; k < 2; ++k) {
            CHECK(cov[k] >= p[k]);                              // coverage
            CHECK(cov[k] - p[k] < th[k] * el[k]);               // minimality
        }
        // the C-ABI computes the same division
        kw_workdiv c{};
        const auto pp = p.padded(), tt = th.padded(), ee = el.padded();
        CHECK(kw_divide_for_gpu(2, pp.data(), tt.data(), ee.data(), &c) == KW_OK);
        CHECK(WorkDiv::fromC(c) == wd);
    }
}

// Acceptance criterion 04 (acceptance.cpp:269-306), same seed, sampler and checks, over every
// backend including GpuCudaRt (whose division the C-ABI must reproduce).
TEST_CASE("criterion 04: work-division law (acceptance.cpp:269-306)")
{
    std::mt19937_64 rng(404);
    const BackendKind backends[] = {BackendKind::Serial, BackendKind::ThreadsParallel, BackendKind::BlocksParallel,
                                    BackendKind::GpuCudaRt};
    auto randomExtent = [&](std::size_t dim, std::size_t maxProduct) {
        std::size_t comp[3] = {1, 1, 1};
        std::size_t budget = maxProduct;
        for (std::size_t k = 0; k < dim; ++k) {
            std::uniform_int_distribution<std::size_t> dist(1, std::max<std::size_t>(1, budget));
            comp[k] = dist(rng);
            budget = std::max<std::size_t>(1, budget / comp[k]);
        }
        return dim == 1 ? IndexVec(comp[0]) : dim == 2 ? IndexVec(comp[0], comp[1]) : IndexVec(comp[0], comp[1], comp[2]);
    };
    std::size_t failures = 0, gpuCases = 0;
    for (int iter = 0; iter < 1000; ++iter) {
        const std::size_t dim = 1 + rng() % 3;
        const IndexVec n = randomExtent(dim, 1 << 20);
        IndexVec b = IndexVec::filled(dim, 1), v = IndexVec::filled(dim, 1);
        for (std::size_t k = 0; k < dim; ++k) {
            b = b.with(k, 1 + rng() % 64);
            v = v.with(k, 1 + rng() % 16);
        }
        const BackendKind backend = backends[rng() % 4];
        const WorkDiv wd = divideForBackend(n, backend, b, v);
        const bool threadLevel = backend == BackendKind::ThreadsParallel || backend == BackendKind::GpuCudaRt;
        if (!threadLevel && wd.threadsPerBlock() != IndexVec::filled(dim, 1))
            ++failures;
        if (threadLevel && wd.threadsPerBlock() != b)
            ++failures;
        const IndexVec coverage = totalExtent(wd, Level::Grid, Unit::Elems);
        for (std::size_t k = 0; k < dim; ++k) {
            if (coverage[k] < n[k])
                ++failures;
            const std::size_t perBlock = wd.threadsPerBlock()[k] * wd.elementsPerThread()[k];
            if ((wd.blocksPerGrid()[k] - 1) * perBlock >= n[k])
                ++failures;
        }
        if (backend == BackendKind::GpuCudaRt) {
            ++gpuCases;
            kw_workdiv c{};
            const auto pp = n.padded(), tt = b.padded(), ee = v.padded();
            if (kw_divide_for_gpu(static_cast<uint32_t>(dim), pp.data(), tt.data(), ee.data(), &c) != KW_OK ||
                !(WorkDiv::fromC(c) == wd))
                ++failures;
        }
    }
    std::printf("  criterion 04: 1000 random (N, B, V), %zu on GpuCudaRt, %zu violations\n", gpuCases, failures);
    CHECK(failures == 0);
}

TEST_CASE("getIdx / getWorkDiv: enum form == template-tag form (test_accel.cpp:61-86)")
{
    const WorkDiv wd(IndexVec(4), IndexVec(16), IndexVec(8));
    const AccContext acc(wd, IndexVec(2), IndexVec(3));
    CHECK(getIdx(acc, Level::Grid, Unit::Threads) == IndexVec(35));
    CHECK((idx::getIdx<Grid, Threads>(acc)) == IndexVec(35));
    CHECK((idx::getIdx<Grid, Threads>(acc)[0u]) == 35u);
    CHECK((idx::getIdx<Grid, Blocks>(acc)) == getIdx(acc, Level::Grid, Unit::Blocks));
    CHECK((idx::getIdx<Block, Threads>(acc)) == getIdx(acc, Level::Block, Unit::Threads));
    CHECK((workdiv::getWorkDiv<Thread, Elems>(acc)[0u]) == 8u);
    const std::pair<Level, Unit> pairs[] = {{Level::Grid, Unit::Blocks},  {Level::Grid, Unit::Threads},
                                            {Level::Grid, Unit::Elems},   {Level::Block, Unit::Threads},
                                            {Level::Block, Unit::Elems},  {Level::Thread, Unit::Elems}};
    const IndexVec tag[] = {workdiv::getWorkDiv<Grid, Blocks>(acc),  workdiv::getWorkDiv<Grid, Threads>(acc),
                            workdiv::getWorkDiv<Grid, Elems>(acc),   workdiv::getWorkDiv<Block, Threads>(acc),
                            workdiv::getWorkDiv<Block, Elems>(acc),  workdiv::getWorkDiv<Thread, Elems>(acc)};
    for (int i = 0; i < 6; ++i)
        CHECK(getWorkDiv(acc, pairs[i].first, pairs[i].second) == tag[i]);
    CHECK_THROWS_AS(getIdx(acc, Level::Thread, Unit::Elems), UsageError);
    const WorkDiv wd3(IndexVec(2, 3, 4), IndexVec(5, 6, 7), IndexVec(1, 1, 1));
    const AccContext a3(wd3, IndexVec(1, 2, 3), IndexVec(4, 5, 6));
    CHECK((idx::getIdx<Grid, Threads>(a3)) == IndexVec(9, 17, 27));
}

TEST_CASE("no CPU back-end in the B200 build")
{
    const WorkDiv wd = kernels::axpyWorkDiv(BackendKind::BlocksParallel, 8, 1, 4);
    CHECK_THROWS_AS(createExec(BackendKind::BlocksParallel, wd, kernels::AxpyKernel{}, kernels::AxpyArgs{}),
                    UsageError);
    CHECK(parseBackend("gpu") == BackendKind::GpuCudaRt);
    CHECK_THROWS_AS(parseBackend("cuda-emulated"), UsageError);
}

// A reference-style functor using the kernel-side services compiles in a host (g++) unit;
// it can only run on the GPU (nvcc + cuda_exec.cuh), so calling the services here throws.
struct HostCompiledReduce {
    void operator()(const AccContext& acc, double* out) const
    {
        double* partial = allocSharedMem<double>(acc, 4);
        partial[0] = 1.0;
        syncBlockThreads(acc);
        atomicAdd(acc, *out, partial[0]);
    }
};

TEST_CASE("host-compiled functors using kernel-side services compile; the services are GPU-only")
{
    kw_workdiv w{1, {1, 1, 1}, {4, 1, 1}, {1, 1, 1}};
    const AccContext acc(w, IndexVec(0), IndexVec(0));
    double out = 0.0;
    CHECK_THROWS_AS(HostCompiledReduce{}(acc, &out), UsageError);
    std::int64_t cell = 0;
    CHECK_THROWS_AS(atomicAdd(acc, cell, std::int64_t{1}), UsageError);
    CHECK_THROWS_AS(syncBlockThreads(acc), UsageError);
}

TEST_CASE("C-ABI usage errors come back as UsageError")
{
    CHECK_THROWS_AS(detail::check(kw_total_extent(nullptr, 0, 0, nullptr)), UsageError);
    CHECK_THROWS_AS(Queue(Device::gpu(4096), QueueFlavor::Sync), UsageError);
}

int main() { return kwcheck::run(); }
