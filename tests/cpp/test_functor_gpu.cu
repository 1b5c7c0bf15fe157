// Generic device functor launch (kernelweave/cuda_exec.cuh): user functors written against the
// reference's kernel-side API run on the GPU. Mirrors acceptance criteria 2 (invocation
// coverage, acceptance.cpp:157-203) and 5 (shared memory + barrier, :358-409) and the atomics
// and index checks of test_accel.cpp:61-86, 151-401.
#include <kernelweave/cuda_exec.cuh>

#include "check.hpp"

#include <cstring>
#include <random>
#include <vector>

using namespace kernelweave;

namespace {
constexpr BackendKind kBk = BackendKind::GpuCudaRt;
const Device kGpu = Device::gpu(0);

template <class T>
std::vector<T> download(const Buffer& d, std::size_t n)
{
    Buffer h(Device::host(), IndexVec(n), sizeof(T));
    Queue q(kGpu, QueueFlavor::Sync);
    copyBuffer(q, h, d, IndexVec(n));
    return std::vector<T>(h.rowData<T>(0), h.rowData<T>(0) + n);
}

template <class T>
Buffer upload(const std::vector<T>& v)
{
    Buffer h(Device::host(), IndexVec(v.size()), sizeof(T));
    std::memcpy(h.rowData<T>(0), v.data(), v.size() * sizeof(T));
    Buffer d(kGpu, IndexVec(v.size()), sizeof(T));
    Queue q(kGpu, QueueFlavor::Sync);
    copyBuffer(q, d, h, h.extent());
    return d;
}
} // namespace

// Every (block, thread) pair runs exactly once: bump a per-grid-thread counter.
struct MarkKernel {
    __device__ void operator()(const AccContext& acc, BufferView counts) const
    {
        const IndexVec gt = idx::getIdx<Grid, Threads>(acc);
        const IndexVec ext = workdiv::getWorkDiv<Grid, Threads>(acc);
        std::size_t lin = 0;
        for (std::size_t k = 0; k < gt.dim(); ++k)
            lin = lin * ext.get(k) + gt.get(k);
        atomicAdd(acc, counts.rowData<std::uint64_t>(0)[lin], std::uint64_t{1});
    }
};
KW_DEVICE_FUNCTOR(MarkKernel)

// Block reduction through allocSharedMem + syncBlockThreads, one atomicAdd per block.
struct BlockReduceKernel {
    static constexpr std::size_t sharedMemBytes = 16 * 1024;
    __device__ void operator()(const AccContext& acc, BufferView out, double value) const
    {
        const std::size_t tpb = getWorkDiv(acc, Level::Block, Unit::Threads).product();
        double* partial = allocSharedMem<double>(acc, tpb);
        const std::size_t t = getIdx(acc, Level::Block, Unit::Threads).get(0);
        if (partial[t] != 0.0) // zero-initialised on first allocation
            atomicAdd(acc, out.rowData<double>(0)[1], 1.0);
        partial[t] = value;
        syncBlockThreads(acc);
        if (t == 0) {
            double s = 0.0;
            for (std::size_t i = 0; i < tpb; ++i)
                s += partial[i];
            atomicAdd(acc, out.rowData<double>(0)[0], s);
        }
    }
};
KW_DEVICE_FUNCTOR(BlockReduceKernel)

// The reference README's functor (AxpyKernel shape), fed BufferViews.
struct ScaleKernel {
    __device__ void operator()(const AccContext& acc, std::size_t n, double alpha, BufferView x, BufferView y) const
    {
        const std::size_t thread = getIdx(acc, Level::Grid, Unit::Threads).get(0);
        const std::size_t chunk = getWorkDiv(acc, Level::Thread, Unit::Elems).get(0);
        const std::size_t first = thread * chunk;
        if (first >= n)
            return;
        const std::size_t count = chunk < n - first ? chunk : n - first;
        const double* xs = x.rowData<double>(0);
        double* ys = y.rowData<double>(0);
        for (std::size_t i = first; i < first + count; ++i)
            ys[i] = __dadd_rn(__dmul_rn(alpha, xs[i]), ys[i]);
    }
};
KW_DEVICE_FUNCTOR(ScaleKernel)

// Both index spellings agree on the device.
struct IndexKernel {
    __device__ void operator()(const AccContext& acc, BufferView out) const
    {
        const IndexVec a = idx::getIdx<Grid, Threads>(acc);
        const IndexVec b = getIdx(acc, Level::Grid, Unit::Threads);
        const IndexVec e = workdiv::getWorkDiv<Grid, Elems>(acc);
        const IndexVec f = getWorkDiv(acc, Level::Grid, Unit::Elems);
        const IndexVec ext = getWorkDiv(acc, Level::Grid, Unit::Threads);
        std::size_t lin = 0;
        for (std::size_t k = 0; k < a.dim(); ++k)
            lin = lin * ext.get(k) + a.get(k);
        out.rowData<std::uint32_t>(0)[lin] = (a == b && e == f) ? 1u : 2u;
    }
};
KW_DEVICE_FUNCTOR(IndexKernel)

// A functor asking for more shared memory than an SM has: its launch fails on the device side.
struct TooMuchSharedKernel {
    static constexpr std::size_t sharedMemBytes = 512 * 1024;
    __device__ void operator()(const AccContext&, BufferView) const {}
};
KW_DEVICE_FUNCTOR(TooMuchSharedKernel)

TEST_CASE("failed tasks are collected, later tasks still run, wait() reports TaskError (queue.hpp:86-93)")
{
    Buffer counts = upload(std::vector<std::uint64_t>(64, 0));
    Queue q(kGpu, QueueFlavor::Async);
    const WorkDiv wd(IndexVec(1), IndexVec(64), IndexVec(1));
    TaskHandle bad1 = q.enqueue(createExec(kBk, wd, TooMuchSharedKernel{}, view(counts)));
    TaskHandle good = q.enqueue(createExec(kBk, wd, MarkKernel{}, view(counts)));
    TaskHandle bad2 = q.enqueue(createExec(kBk, wd, TooMuchSharedKernel{}, view(counts)));
    bool threw = false;
    std::size_t failed = 0;
    try {
        q.wait();
    }
    catch (const TaskError& e) {
        threw = true;
        failed = e.failedCount();
    }
    CHECK(threw);
    CHECK(failed == 2);
    CHECK(bad1.state() == TaskState::Failed);
    CHECK(bad2.state() == TaskState::Failed);
    CHECK(good.state() == TaskState::Done);
    const auto got = download<std::uint64_t>(counts, 64);
    bool ok = true;
    for (auto v : got)
        ok = ok && v == 1; // the task between the failures ran
    CHECK(ok);
    q.wait(); // failures were reported once; the queue is clean again
}

TEST_CASE("invocation coverage: every (block, thread) exactly once (acceptance crit. 2)")
{
    std::mt19937_64 rng(202);
    for (int iter = 0; iter < 12; ++iter) {
        const std::size_t dim = 1 + iter % 3;
        auto r = [&](std::size_t lo, std::size_t hi) { return lo + rng() % (hi - lo + 1); };
        const WorkDiv wd = dim == 1 ? WorkDiv(IndexVec(r(1, 300)), IndexVec(r(1, 256)), IndexVec(r(1, 3)))
                           : dim == 2 ? WorkDiv(IndexVec(r(1, 40), r(1, 40)), IndexVec(r(1, 16), r(1, 32)), IndexVec(1, 2))
                                      : WorkDiv(IndexVec(r(1, 6), r(1, 6), r(1, 6)), IndexVec(r(1, 4), r(1, 8), r(1, 16)),
                                                IndexVec(1, 1, 1));
        const std::size_t n = totalExtent(wd, Level::Grid, Unit::Threads).product();
        Buffer counts = upload(std::vector<std::uint64_t>(n, 0));
        executeTask(kBk, wd, MarkKernel{}, view(counts));
        const auto got = download<std::uint64_t>(counts, n);
        bool ok = true;
        for (auto v : got)
            ok = ok && v == 1;
        CHECK(ok);
    }
}

TEST_CASE("shared memory zeroed, barrier, atomics (acceptance crit. 5, test_accel.cpp:365-401)")
{
    Buffer out = upload(std::vector<double>{0.0, 0.0});
    // 64 blocks x 64 threads, each thread contributes 0.5 -> 2048.0
    executeTask(kBk, WorkDiv(IndexVec(64), IndexVec(64), IndexVec(1)), BlockReduceKernel{}, view(out), 0.5);
    const auto got = download<double>(out, 2);
    CHECK(got[0] == 2048.0);
    CHECK(got[1] == 0.0); // no thread saw a non-zero fresh allocation
}

TEST_CASE("README functor runs unchanged on the GPU, bitwise equal to axpyReference")
{
    const std::size_t n = 1 << 20;
    std::mt19937_64 rng(42);
    std::vector<double> x(n), y(n);
    for (auto* v : {&x, &y})
        for (auto& e : *v)
            e = static_cast<double>(rng() >> 11) * 0x1.0p-53 * 10.0;
    std::vector<double> want = y;
    for (std::size_t i = 0; i < n; ++i)
        want[i] = 2.5 * x[i] + want[i];
    Buffer dx = upload(x), dy = upload(y);
    executeTask(kBk, divideForBackend(IndexVec(n), kBk, IndexVec(256), IndexVec(4)), ScaleKernel{}, n, 2.5, view(dx),
                view(dy));
    const auto got = download<double>(dy, n);
    std::size_t bad = 0, first = n;
    for (std::size_t i = 0; i < n; ++i)
        if (got[i] != want[i]) {
            if (first == n)
                first = i;
            ++bad;
        }
    if (bad)
        std::printf("  %zu mismatches, first at %zu: got %.17g want %.17g (x %.17g y %.17g)\n", bad, first,
                    got[first], want[first], x[first], y[first]);
    CHECK(bad == 0);
}

TEST_CASE("index spellings agree on the device (test_accel.cpp:61-86)")
{
    const WorkDiv wd(IndexVec(3, 5, 7), IndexVec(2, 4, 8), IndexVec(1, 2, 3));
    const std::size_t n = totalExtent(wd, Level::Grid, Unit::Threads).product();
    Buffer out = upload(std::vector<std::uint32_t>(n, 0));
    Queue q(kGpu, QueueFlavor::Async);
    q.enqueue(createExec(kBk, wd, IndexKernel{}, view(out)));
    q.wait();
    const auto got = download<std::uint32_t>(out, n);
    bool ok = true;
    for (auto v : got)
        ok = ok && v == 1;
    CHECK(ok);
    CHECK_THROWS_AS(createExec(kBk, WorkDiv(IndexVec(1), IndexVec(2048), IndexVec(1)), IndexKernel{}, view(out)),
                    UsageError);
}

int main()
{
    if (deviceCount() == 0) {
        std::printf("no CUDA device\n");
        return 2;
    }
    return kwcheck::run();
}
