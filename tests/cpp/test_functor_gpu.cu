// Generic device functor launch (kernelweave/cuda_exec.cuh): user functors written against the
// reference's kernel-side API run on the GPU. Mirrors acceptance criteria 2 (invocation
// coverage, acceptance.cpp:157-203) and 5 (shared memory + barrier, :358-409) and the atomics
// and index checks of test_accel.cpp:61-86, 151-401.
#include <kernelweave/cuda_exec.cuh>

#include "check.hpp"

#include <algorithm>
#include <array>
#include <atomic>
#include <thread>
#include <cmath>
#include <chrono>
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

// allocSharedMem past the block's declared arena: the reference throws UsageError out of
// operator() (accel.cpp:286-292); here the block retires and the task fails (no trap).
struct SharedOverflowKernel {
    static constexpr std::size_t sharedMemBytes = 1024;
    __device__ void operator()(const AccContext& acc, BufferView out) const
    {
        double* a = allocSharedMem<double>(acc, 64);  // 512 B: fits
        double* b = allocSharedMem<double>(acc, 128); // 1 KiB more: past the 1 KiB arena
        a[0] = b[0] = 1.0;                            // never reached
        atomicAdd(acc, out.rowData<std::uint64_t>(0)[0], std::uint64_t{1});
    }
};
KW_DEVICE_FUNCTOR(SharedOverflowKernel)

// test_accel.cpp:403-430: the functor "throws" in block 3 — on the GPU, failTask + return.
struct FailKernel {
    __device__ void operator()(const AccContext& acc, unsigned code) const
    {
        const IndexVec b = idx::getIdx<Grid, Blocks>(acc);
        if (b.get(0) == 3) {
            failTask(acc, code);
            return;
        }
    }
};
KW_DEVICE_FUNCTOR(FailKernel)

// test_accel.cpp:111-127 / 365-401: int64, f64 and u64 atomics from a 256 x 16 grid.
struct IncKernel {
    __device__ void operator()(const AccContext& acc, BufferView cells) const
    {
        atomicAdd(acc, cells.rowData<std::int64_t>(0)[0], std::int64_t{1});
        atomicAdd(acc, cells.rowData<double>(0)[1], 0.5);
        atomicAdd(acc, cells.rowData<std::uint64_t>(0)[2], std::uint64_t{2});
    }
};
KW_DEVICE_FUNCTOR(IncKernel)

// Adding zero returns the old value and leaves the cell unchanged (test_accel.cpp:389-400).
struct ZeroAddKernel {
    __device__ void operator()(const AccContext& acc, BufferView cell, BufferView old) const
    {
        old.rowData<double>(0)[0] = atomicAdd(acc, cell.rowData<double>(0)[0], 0.0);
    }
};
KW_DEVICE_FUNCTOR(ZeroAddKernel)

// test_accel.cpp:151-170: two successive allocations are zeroed and disjoint.
struct TwoAllocKernel {
    __device__ void operator()(const AccContext& acc, BufferView out) const
    {
        double* first = allocSharedMem<double>(acc, 16);
        double* second = allocSharedMem<double>(acc, 16);
        bool zeroed = true;
        for (int i = 0; i < 16; ++i)
            zeroed = zeroed && first[i] == 0.0 && second[i] == 0.0;
        const bool disjoint = (first + 16 <= second) || (second + 16 <= first);
        const std::size_t b = idx::getIdx<Grid, Blocks>(acc).get(0);
        const std::size_t t = idx::getIdx<Block, Threads>(acc).get(0);
        out.rowData<std::int64_t>(0)[2 * (b * 32 + t)] = zeroed ? 1 : 0;
        out.rowData<std::int64_t>(0)[2 * (b * 32 + t) + 1] = disjoint ? 1 : 0;
    }
};
KW_DEVICE_FUNCTOR(TwoAllocKernel)

// test_accel.cpp:172-196 + 198-244: thread 0 writes a block-unique token, the barrier publishes
// it to every thread of the block, and no other (concurrently resident) block disturbs it.
struct AliasKernel {
    static constexpr std::size_t sharedMemBytes = 1024;
    __device__ void operator()(const AccContext& acc, BufferView out) const
    {
        double* shared = allocSharedMem<double>(acc, 64);
        const std::size_t b = idx::getIdx<Grid, Blocks>(acc).get(0);
        const std::size_t t = idx::getIdx<Block, Threads>(acc).get(0);
        if (t == 0)
            for (int i = 0; i < 64; ++i)
                shared[i] = static_cast<double>(b * 64 + i);
        syncBlockThreads(acc);
        double sink = 0.0;
        for (int spin = 0; spin < 2000; ++spin)
            sink += shared[spin % 64];
        bool intact = sink >= 0.0;
        for (int i = 0; i < 64; ++i)
            intact = intact && shared[i] == static_cast<double>(b * 64 + i);
        out.rowData<std::int64_t>(0)[b * 8 + t] = intact ? 1 : 0;
    }
};
KW_DEVICE_FUNCTOR(AliasKernel)

// test_accel.cpp:300-341: staged power-of-two tree reduction, one barrier per stage.
struct TreeReduceKernel {
    __device__ void operator()(const AccContext& acc, BufferView in, BufferView out, std::size_t n) const
    {
        const std::size_t threads = getWorkDiv(acc, Level::Block, Unit::Threads).get(0);
        const std::size_t t = getIdx(acc, Level::Block, Unit::Threads).get(0);
        std::int64_t* partial = allocSharedMem<std::int64_t>(acc, threads);
        const std::int64_t* data = in.rowData<std::int64_t>(0);
        std::int64_t local = 0;
        for (std::size_t i = t; i < n; i += threads)
            local += data[i];
        partial[t] = local;
        syncBlockThreads(acc);
        for (std::size_t stride = threads / 2; stride > 0; stride /= 2) {
            if (t < stride)
                partial[t] += partial[t + stride];
            syncBlockThreads(acc);
        }
        if (t == 0)
            out.rowData<std::int64_t>(0)[0] = partial[0];
    }
};
KW_DEVICE_FUNCTOR(TreeReduceKernel)

struct EmptyKernel {
    __device__ void operator()(const AccContext&) const {}
};
KW_DEVICE_FUNCTOR(EmptyKernel)

TEST_CASE("kernel failure fails the task; later tasks still run (test_accel.cpp:403-430, queue.hpp:86-93)")
{
    // executeTask (synchronous) surfaces it as TaskError
    bool threw = false;
    try {
        executeTask(kBk, WorkDiv(IndexVec(8), IndexVec(32), IndexVec(1)), FailKernel{}, 7u);
    }
    catch (const TaskError& e) {
        threw = e.failedCount() == 1 && std::string(e.what()).find("code 7") != std::string::npos;
    }
    CHECK(threw);
    // Async: two failing tasks around a good one; handles, count, and a clean second wait
    Buffer counts = upload(std::vector<std::uint64_t>(64, 0));
    Queue q(kGpu, QueueFlavor::Async);
    TaskHandle bad1 = q.enqueue(createExec(kBk, WorkDiv(IndexVec(4), IndexVec(16), IndexVec(1)), FailKernel{}, 3u));
    TaskHandle good = q.enqueue(createExec(kBk, WorkDiv(IndexVec(1), IndexVec(64), IndexVec(1)), MarkKernel{},
                                           view(counts)));
    TaskHandle bad2 = q.enqueue(createExec(kBk, WorkDiv(IndexVec(4), IndexVec(16), IndexVec(1)), FailKernel{}, 5u));
    std::size_t failed = 0;
    try {
        q.wait();
    }
    catch (const TaskError& e) {
        failed = e.failedCount();
    }
    CHECK(failed == 2);
    CHECK(bad1.state() == TaskState::Failed);
    CHECK(bad1.error() != nullptr);
    CHECK(bad2.state() == TaskState::Failed);
    CHECK(good.state() == TaskState::Done);
    const auto got = download<std::uint64_t>(counts, 64);
    bool ok = true;
    for (auto v : got)
        ok = ok && v == 1;
    CHECK(ok);
    q.wait();
    // a task without the failing block succeeds
    TaskHandle fine = q.enqueue(createExec(kBk, WorkDiv(IndexVec(3), IndexVec(16), IndexVec(1)), FailKernel{}, 9u));
    q.wait();
    CHECK(fine.state() == TaskState::Done);
}

TEST_CASE("a 256x16 grid performs 4096 invocations; atomics int64/f64/u64 (test_accel.cpp:111-127, 365-401)")
{
    Buffer cells = upload(std::vector<std::uint64_t>(3, 0));
    executeTask(kBk, WorkDiv(IndexVec(256), IndexVec(16), IndexVec(1)), IncKernel{}, view(cells));
    const auto got = download<std::uint64_t>(cells, 3);
    double f = 0.0;
    std::memcpy(&f, &got[1], 8);
    CHECK(got[0] == 4096);
    CHECK(f == 2048.0);
    CHECK(got[2] == 8192);
    Buffer cell = upload(std::vector<double>{123.5});
    Buffer old = upload(std::vector<double>{0.0});
    executeTask(kBk, WorkDiv(IndexVec(1), IndexVec(1), IndexVec(1)), ZeroAddKernel{}, view(cell), view(old));
    CHECK(download<double>(cell, 1)[0] == 123.5);
    CHECK(download<double>(old, 1)[0] == 123.5);
}

TEST_CASE("empty kernel completes without effect (test_accel.cpp:101-109)")
{
    executeTask(kBk, WorkDiv(IndexVec(2, 2), IndexVec(1, 2), IndexVec(1, 1)), EmptyKernel{});
    CHECK(true);
}

TEST_CASE("shared memory: successive allocations zeroed and disjoint; blocks never alias (test_accel.cpp:151-244)")
{
    Buffer out = upload(std::vector<std::int64_t>(2 * 4 * 32, 0));
    executeTask(kBk, WorkDiv(IndexVec(4), IndexVec(32), IndexVec(1)), TwoAllocKernel{}, view(out));
    bool ok = true;
    for (auto v : download<std::int64_t>(out, 2 * 4 * 32))
        ok = ok && v == 1;
    CHECK(ok);
    const std::size_t blocks = 592; // four resident waves' worth on 148 SMs
    Buffer alias = upload(std::vector<std::int64_t>(blocks * 8, 0));
    executeTask(kBk, WorkDiv(IndexVec(blocks), IndexVec(8), IndexVec(1)), AliasKernel{}, view(alias));
    ok = true;
    for (auto v : download<std::int64_t>(alias, blocks * 8))
        ok = ok && v == 1;
    CHECK(ok);
}

TEST_CASE("staged shared-memory reduction matches the sequential sum (test_accel.cpp:322-341)")
{
    std::mt19937_64 rng(314);
    for (std::size_t threads : {2u, 4u, 8u, 16u, 256u, 1024u}) {
        for (int iter = 0; iter < 5; ++iter) {
            const std::size_t n = 1 + rng() % (1u << 14);
            std::vector<std::int64_t> v(n);
            std::int64_t expected = 0;
            for (auto& e : v) {
                e = static_cast<std::int64_t>(rng() % 1000) - 500;
                expected += e;
            }
            Buffer in = upload(v);
            Buffer out = upload(std::vector<std::int64_t>{0});
            executeTask(kBk, WorkDiv(IndexVec(1), IndexVec(threads), IndexVec(1)), TreeReduceKernel{}, view(in),
                        view(out), n);
            CHECK(download<std::int64_t>(out, 1)[0] == expected);
        }
    }
}

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

TEST_CASE("allocSharedMem overflow fails the task, not the context; later tasks run (accel.cpp:286-292)")
{
    Buffer out = upload(std::vector<std::uint64_t>(64, 0));
    Queue q(kGpu, QueueFlavor::Async);
    TaskHandle bad = q.enqueue(createExec(kBk, WorkDiv(IndexVec(8), IndexVec(32), IndexVec(1)),
                                          SharedOverflowKernel{}, view(out)));
    TaskHandle good = q.enqueue(createExec(kBk, WorkDiv(IndexVec(1), IndexVec(64), IndexVec(1)), MarkKernel{},
                                           view(out)));
    std::string msg;
    std::size_t failed = 0;
    try {
        q.wait();
    }
    catch (const TaskError& e) {
        failed = e.failedCount();
        msg = e.what();
    }
    CHECK(failed == 1);
    CHECK(msg.find("allocSharedMem") != std::string::npos);
    CHECK(bad.state() == TaskState::Failed);
    CHECK(good.state() == TaskState::Done);
    const auto got = download<std::uint64_t>(out, 64);
    bool ok = got[0] == 1; // slot 0: MarkKernel's 1, never the overflow kernel's atomicAdd
    for (std::size_t i = 1; i < 64; ++i)
        ok = ok && got[i] == 1;
    CHECK(ok);
    // the context is healthy: a fresh synchronous task runs
    executeTask(kBk, WorkDiv(IndexVec(1), IndexVec(64), IndexVec(1)), MarkKernel{}, view(out));
    CHECK(download<std::uint64_t>(out, 64)[5] == 2);
}

TEST_CASE("a generic functor enqueue on a shut-down queue is a UsageError (queue.cpp enqueueBody)")
{
    Buffer out = upload(std::vector<std::uint64_t>(64, 0));
    Queue q(kGpu, QueueFlavor::Async);
    q.shutdown();
    CHECK_THROWS_AS(q.enqueue(createExec(kBk, WorkDiv(IndexVec(1), IndexVec(64), IndexVec(1)), MarkKernel{},
                                         view(out))),
                    UsageError);
    CHECK(download<std::uint64_t>(out, 64)[0] == 0);
}

TEST_CASE("concurrent enqueue and wait: every device-side failure is counted exactly once (queue.hpp:86-93)")
{
    // Thread A enqueues failing functors while thread B drains the queue in a loop. A failure
    // slot may only be resolved by a drain that started after its kernel was in the stream;
    // a slot resolved early would be recycled unread and its failure lost.
    Queue q(kGpu, QueueFlavor::Async);
    constexpr int kTasks = 400;
    std::atomic<bool> done{false};
    std::atomic<std::size_t> seen{0};
    std::thread waiter([&] {
        while (!done.load()) {
            try {
                q.wait();
            }
            catch (const TaskError& e) {
                seen += e.failedCount();
            }
        }
    });
    for (int i = 0; i < kTasks; ++i)
        q.enqueue(createExec(kBk, WorkDiv(IndexVec(8), IndexVec(32), IndexVec(1)), FailKernel{}, 1u + i % 7));
    done = true;
    waiter.join();
    try {
        q.wait();
    }
    catch (const TaskError& e) {
        seen += e.failedCount();
    }
    std::printf("  %d failing tasks, %zu failures reported\n", kTasks, seen.load());
    CHECK(seen.load() == kTasks);
}

// The shipped functors' operator() composed inside user device functors (verdict r1: "code
// that invokes or composes the functor directly"): bitwise equal to the library's own launches.
struct ComposedAxpy {
    __device__ void operator()(const AccContext& acc, kernels::AxpyArgsView<float> a) const
    {
        kernels::AxpyKernel{}(acc, a);
    }
};
KW_DEVICE_FUNCTOR(ComposedAxpy)
struct ComposedNaive {
    __device__ void operator()(const AccContext& acc, kernels::GemmArgsView g) const { kernels::GemmNaiveKernel{}(acc, g); }
};
KW_DEVICE_FUNCTOR(ComposedNaive)
struct ComposedTiled {
    static constexpr std::size_t sharedMemBytes = 3 * 16 * 16 * sizeof(double);
    __device__ void operator()(const AccContext& acc, kernels::GemmArgsView g) const { kernels::GemmTiledKernel{}(acc, g); }
};
KW_DEVICE_FUNCTOR(ComposedTiled)

TEST_CASE("AxpyKernel / GemmNaiveKernel / GemmTiledKernel operator() compose in device functors, bit-exact")
{
    std::mt19937_64 rng(77);
    const std::size_t n = 1000003;
    std::vector<float> xv(n), yv(n);
    for (std::size_t i = 0; i < n; ++i) {
        xv[i] = static_cast<float>((rng() >> 11) * 0x1.0p-53 * 10.0);
        yv[i] = static_cast<float>((rng() >> 11) * 0x1.0p-53 * 10.0);
    }
    Buffer x = upload(xv), y1 = upload(yv), y2 = upload(yv);
    executeTask(kBk, kernels::axpyWorkDiv(kBk, n, 256, 8), kernels::AxpyKernel{},
                kernels::AxpyArgsF32{n, 2.75f, &x, &y1});
    executeTask(kBk, kernels::axpyWorkDiv(kBk, n, 256, 8), ComposedAxpy{},
                kernels::toView(kernels::AxpyArgsF32{n, 2.75f, &x, &y2}));
    const auto a1 = download<float>(y1, n), a2 = download<float>(y2, n);
    std::size_t bad = 0, first = n;
    for (std::size_t i = 0; i < n; ++i)
        if (std::memcmp(&a1[i], &a2[i], 4) != 0 && bad++ == 0)
            first = i;
    if (bad) {
        volatile float p = 2.75f * xv[first];
        std::printf("  composed AXPY: %zu mismatches, first %zu: x %a y0 %a tuned %a composed %a host %a\n", bad, first,
                    xv[first], yv[first], a1[first], a2[first], p + yv[first]);
    }
    CHECK(bad == 0);

    for (auto [m, nn, k] : {std::array<std::size_t, 3>{1, 1, 1}, {37, 29, 41}, {130, 67, 200}, {64, 64, 64}}) {
        auto mat = [&](std::size_t r, std::size_t c) {
            std::vector<double> v(r * c);
            for (auto& e : v)
                e = (rng() >> 11) * 0x1.0p-53 * 10.0;
            Buffer h(Device::host(), IndexVec(r, c), 8);
            for (std::size_t i = 0; i < r; ++i)
                std::memcpy(h.rowData<double>(i), v.data() + i * c, c * 8);
            Buffer d(kGpu, IndexVec(r, c), 8);
            Queue q(kGpu, QueueFlavor::Sync);
            copyBuffer(q, d, h, h.extent());
            return d;
        };
        Buffer A = mat(m, k), B = mat(k, nn), C0 = mat(m, nn);
        auto fresh = [&] {
            Buffer c(kGpu, IndexVec(m, nn), 8);
            Queue q(kGpu, QueueFlavor::Sync);
            copyBuffer(q, c, C0, C0.extent());
            return c;
        };
        auto rows = [&](const Buffer& c) {
            Buffer h(Device::host(), c.extent(), 8);
            Queue q(kGpu, QueueFlavor::Sync);
            copyBuffer(q, h, c, c.extent());
            std::vector<double> out(m * nn);
            for (std::size_t i = 0; i < m; ++i)
                std::memcpy(out.data() + i * nn, h.rowData<double>(i), nn * 8);
            return out;
        };
        Buffer cRef = fresh(), cNaive = fresh(), cTiled = fresh();
        const kernels::GemmArgs ref{m, nn, k, 1.25, 0.5, &A, &B, &cRef};
        executeTask(kBk, kernels::gemmNaiveWorkDiv(kBk, m, nn, 4, 4), kernels::GemmNaiveKernel{}, ref);
        executeTask(kBk, kernels::gemmNaiveWorkDiv(BackendKind::ThreadsParallel, m, nn, 8, 3), ComposedNaive{},
                    kernels::toView(kernels::GemmArgs{m, nn, k, 1.25, 0.5, &A, &B, &cNaive}));
        kernels::GemmArgs tg{m, nn, k, 1.25, 0.5, &A, &B, &cTiled};
        tg.tile = 16;
        executeTask(kBk, kernels::gemmTiledWorkDiv(BackendKind::ThreadsParallel, m, nn, 16), ComposedTiled{},
                    kernels::toView(tg));
        const auto want = rows(cRef);
        CHECK(want == rows(cNaive));
        CHECK(std::memcmp(want.data(), rows(cTiled).data(), want.size() * 8) == 0);
    }
}

// Acceptance criterion 03 (acceptance.cpp:205-267) on the device linearisation every functor
// launch uses (detail::logicalBlockIdx): every extent of dims 1-3 with product <= 10^4, each box
// walked in row-major order by nested loops; the device's logical block for walk position `lin`
// must be the walked index (a bijection onto [0, product) in the reference's order). Same
// extent set, same point count as the reference: 3,263,713,235.
__global__ void criterion03Kernel(const unsigned long long* ext, std::size_t nExt, unsigned long long* counters)
{
    unsigned long long points = 0, failures = 0;
    for (std::size_t e = blockIdx.x; e < nExt; e += gridDim.x) {
        const unsigned dim = static_cast<unsigned>(ext[4 * e + 3]);
        const std::size_t a = ext[4 * e], b = ext[4 * e + 1], c = ext[4 * e + 2];
        kw_workdiv wd{};
        wd.dim = dim;
        for (int k = 0; k < 3; ++k)
            wd.blocks[k] = wd.threads[k] = wd.elems[k] = 1;
        wd.blocks[0] = a;
        if (dim >= 2)
            wd.blocks[1] = b;
        if (dim == 3)
            wd.blocks[2] = c;
        if (kernelweave::detail::logicalBlockCount(wd) != a * b * c)
            ++failures;
        for (std::size_t i0 = threadIdx.x; i0 < a; i0 += blockDim.x) {
            std::size_t lin = i0 * b * c;
            for (std::size_t i1 = 0; i1 < b; ++i1)
                for (std::size_t i2 = 0; i2 < c; ++i2, ++lin) {
                    const IndexVec walk = dim == 1 ? IndexVec(i0) : dim == 2 ? IndexVec(i0, i1) : IndexVec(i0, i1, i2);
                    if (kernelweave::detail::logicalBlockIdx(wd, lin) != walk)
                        ++failures;
                    ++points;
                }
        }
    }
    atomicAdd(&counters[0], points);
    atomicAdd(&counters[1], failures);
}

TEST_CASE("criterion 03 on the device: exhaustive logical-block linearisation (acceptance.cpp:205-267)")
{
    const std::size_t cap = 10000;
    std::vector<unsigned long long> ext;
    for (std::size_t a = 1; a <= cap; ++a)
        ext.insert(ext.end(), {a, 1, 1, 1});
    for (std::size_t a = 1; a <= cap; ++a)
        for (std::size_t b = 1; a * b <= cap; ++b)
            ext.insert(ext.end(), {a, b, 1, 2});
    for (std::size_t a = 1; a <= cap; ++a)
        for (std::size_t b = 1; a * b <= cap; ++b)
            for (std::size_t c = 1; a * b * c <= cap; ++c)
                ext.insert(ext.end(), {a, b, c, 3});
    const std::size_t nExt = ext.size() / 4;
    unsigned long long *dExt = nullptr, *dCnt = nullptr;
    CHECK(cudaMalloc(&dExt, ext.size() * 8) == cudaSuccess);
    CHECK(cudaMalloc(&dCnt, 16) == cudaSuccess);
    cudaMemcpy(dExt, ext.data(), ext.size() * 8, cudaMemcpyHostToDevice);
    cudaMemset(dCnt, 0, 16);
    const auto t0 = std::chrono::steady_clock::now();
    criterion03Kernel<<<148 * 8, 256>>>(dExt, nExt, dCnt);
    CHECK(cudaDeviceSynchronize() == cudaSuccess);
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    unsigned long long cnt[2] = {};
    cudaMemcpy(cnt, dCnt, 16, cudaMemcpyDeviceToHost);
    cudaFree(dExt);
    cudaFree(dCnt);
    std::printf("  criterion 03 (device): %zu extents, %llu points, %llu failures, %.2f s\n", nExt, cnt[0], cnt[1], s);
    CHECK(cnt[0] == 3263713235ull);
    CHECK(cnt[1] == 0);
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

TEST_CASE("logical grids far larger than resident, and past CUDA's 65535 grid limit, run each pair once")
{
    for (const WorkDiv& wd : {WorkDiv(IndexVec(100000), IndexVec(64), IndexVec(1)),
                              WorkDiv(IndexVec(70000, 3), IndexVec(2, 16), IndexVec(1, 1)),
                              WorkDiv(IndexVec(3, 70001, 2), IndexVec(1, 2, 8), IndexVec(1, 1, 1))}) {
        const std::size_t n = totalExtent(wd, Level::Grid, Unit::Threads).product();
        Buffer counts = upload(std::vector<std::uint64_t>(n, 0));
        executeTask(kBk, wd, MarkKernel{}, view(counts));
        const auto got = download<std::uint64_t>(counts, n);
        bool ok = true;
        for (auto v : got)
            ok = ok && v == 1;
        CHECK(ok);
    }
    // shared-arena reuse across the logical blocks one CUDA block walks
    const std::size_t blocks = 50000;
    Buffer alias = upload(std::vector<std::int64_t>(blocks * 8, 0));
    executeTask(kBk, WorkDiv(IndexVec(blocks), IndexVec(8), IndexVec(1)), AliasKernel{}, view(alias));
    bool ok = true;
    for (auto v : download<std::int64_t>(alias, blocks * 8))
        ok = ok && v == 1;
    CHECK(ok);
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

// The paper's DGEMM evaluation: the CUDA programming guide's shared-memory
// tiled DGEMM (§3.2.3, 16 x 16 tiles, one output per thread) translated one-to-one into a
// kernelweave functor, against the same algorithm written natively in CUDA.
constexpr int kPaperTile = 16;

struct PaperTiledGemm {
    static constexpr std::size_t sharedMemBytes = 2 * kPaperTile * kPaperTile * sizeof(double);
    __device__ void operator()(const AccContext& acc, std::size_t n, BufferView a, BufferView b, BufferView c) const
    {
        double* sa = allocSharedMem<double>(acc, kPaperTile * kPaperTile);
        double* sb = allocSharedMem<double>(acc, kPaperTile * kPaperTile);
        const IndexVec blk = idx::getIdx<Grid, Blocks>(acc);
        const IndexVec thr = idx::getIdx<Block, Threads>(acc);
        const std::size_t ty = thr.get(0), tx = thr.get(1);
        const std::size_t row = blk.get(0) * kPaperTile + ty, col = blk.get(1) * kPaperTile + tx;
        const double* A = a.rowData<double>(0);
        const double* B = b.rowData<double>(0);
        const std::size_t lda = a.leadingDim<double>(), ldb = b.leadingDim<double>();
        double sum = 0.0;
        for (std::size_t k0 = 0; k0 < n; k0 += kPaperTile) {
            sa[ty * kPaperTile + tx] = row < n && k0 + tx < n ? A[row * lda + k0 + tx] : 0.0;
            sb[ty * kPaperTile + tx] = k0 + ty < n && col < n ? B[(k0 + ty) * ldb + col] : 0.0;
            syncBlockThreads(acc);
            for (int p = 0; p < kPaperTile; ++p)
                sum = __dadd_rn(sum, __dmul_rn(sa[ty * kPaperTile + p], sb[p * kPaperTile + tx]));
            syncBlockThreads(acc);
        }
        if (row < n && col < n)
            c.rowData<double>(row)[col] = sum;
    }
};
KW_DEVICE_FUNCTOR(PaperTiledGemm)

__global__ void native_paper_tiled_gemm(std::size_t n, const double* A, std::size_t lda, const double* B,
                                        std::size_t ldb, double* C, std::size_t ldc)
{
    __shared__ double sa[kPaperTile][kPaperTile];
    __shared__ double sb[kPaperTile][kPaperTile];
    const std::size_t ty = threadIdx.y, tx = threadIdx.x;
    const std::size_t row = blockIdx.y * kPaperTile + ty, col = blockIdx.x * kPaperTile + tx;
    double sum = 0.0;
    for (std::size_t k0 = 0; k0 < n; k0 += kPaperTile) {
        sa[ty][tx] = row < n && k0 + tx < n ? A[row * lda + k0 + tx] : 0.0;
        sb[ty][tx] = k0 + ty < n && col < n ? B[(k0 + ty) * ldb + col] : 0.0;
        __syncthreads();
        for (int p = 0; p < kPaperTile; ++p)
            sum = __dadd_rn(sum, __dmul_rn(sa[ty][p], sb[p][tx]));
        __syncthreads();
    }
    if (row < n && col < n)
        C[row * ldc + col] = sum;
}

TEST_CASE("paper's one-to-one tiled DGEMM: functor vs native CUDA, same bits, >= 94 % relative speed (PAPER.md:658-671)")
{
    for (std::size_t n : {1024u, 2048u}) {
        std::vector<double> av(n * n), bv(n * n);
        std::mt19937_64 rng(n);
        for (auto* v : {&av, &bv})
            for (auto& e : *v)
                e = static_cast<double>(rng() >> 11) * 0x1.0p-53;
        Buffer a2(kGpu, IndexVec(n, n), 8), b2(kGpu, IndexVec(n, n), 8), c1(kGpu, IndexVec(n, n), 8),
            c2(kGpu, IndexVec(n, n), 8);
        // pitched 2-D operands filled from the dense vectors
        Buffer ha(Device::host(), IndexVec(n, n), 8), hb(Device::host(), IndexVec(n, n), 8);
        for (std::size_t r = 0; r < n; ++r) {
            std::memcpy(ha.rowData<double>(r), av.data() + r * n, n * 8);
            std::memcpy(hb.rowData<double>(r), bv.data() + r * n, n * 8);
        }
        Queue q(kGpu, QueueFlavor::Sync);
        copyBuffer(q, a2, ha, ha.extent());
        copyBuffer(q, b2, hb, hb.extent());
        const WorkDiv wd(IndexVec(n / kPaperTile, n / kPaperTile), IndexVec(kPaperTile, kPaperTile), IndexVec(1, 1));
        auto median_ms = [](auto&& run) {
            run();
            std::vector<double> t;
            for (int r = 0; r < 7; ++r) {
                const auto t0 = std::chrono::steady_clock::now();
                run();
                t.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
            }
            std::sort(t.begin(), t.end());
            return t[3];
        };
        const double functor = median_ms([&] { executeTask(kBk, wd, PaperTiledGemm{}, n, view(a2), view(b2), view(c1)); });
        void* sp = nullptr;
        kw_queue_stream(q.native(), &sp);
        const double native = median_ms([&] {
            native_paper_tiled_gemm<<<dim3(n / kPaperTile, n / kPaperTile), dim3(kPaperTile, kPaperTile), 0,
                                      static_cast<cudaStream_t>(sp)>>>(n, a2.rowData<double>(0), a2.leadingDim<double>(),
                                                                       b2.rowData<double>(0), b2.leadingDim<double>(),
                                                                       c2.rowData<double>(0), c2.leadingDim<double>());
            q.wait();
        });
        Buffer o1(Device::host(), IndexVec(n, n), 8), o2(Device::host(), IndexVec(n, n), 8);
        copyBuffer(q, o1, c1, c1.extent());
        copyBuffer(q, o2, c2, c2.extent());
        bool same = true;
        for (std::size_t r = 0; r < n && same; ++r)
            same = std::memcmp(o1.rowData<double>(r), o2.rowData<double>(r), n * 8) == 0;
        std::printf("  paper tiled DGEMM n=%zu: functor %.3f ms, native %.3f ms -> relative performance %.1f %%\n", n,
                    functor, native, 100.0 * native / functor);
        CHECK(same);
        CHECK(native / functor >= 0.94); // the paper reports >= 94 % for this translation on K20
    }
}

// The paper's performance-portability experiment: ONE single-source tiled
// DGEMM kernel using every level of the hierarchy — grid of blocks, 16 x 16 threads per block,
// E x E elements per thread (getWorkDiv<Thread, Elems>), shared-memory tiles — measured against
// the architecture's FP64 peak (≈ 20 % on K20/K80/Xeon/Opteron in the paper).
template <int E>
struct PaperHierarchicalGemm {
    static constexpr int T = 16, BK = 16, BM = T * E;
    static constexpr std::size_t sharedMemBytes = static_cast<std::size_t>(2 * BM * (BK + 1)) * sizeof(double);
    __device__ void operator()(const AccContext& acc, std::size_t n, double alpha, double beta, BufferView a,
                               BufferView b, BufferView c) const
    {
        const IndexVec elems = workdiv::getWorkDiv<Thread, Elems>(acc); // (E, E) by construction
        const IndexVec blk = idx::getIdx<Grid, Blocks>(acc);
        const IndexVec thr = idx::getIdx<Block, Threads>(acc);
        if (elems.get(0) != static_cast<std::size_t>(E) || elems.get(1) != static_cast<std::size_t>(E)) {
            failTask(acc, 1);
            return;
        }
        double* sa = allocSharedMem<double>(acc, BM * (BK + 1)); // [BM][BK+1], padded
        double* sb = allocSharedMem<double>(acc, BK * (BM + 1)); // [BK][BN+1]
        const int ty = static_cast<int>(thr.get(0)), tx = static_cast<int>(thr.get(1)), tid = ty * T + tx;
        const std::size_t row0 = blk.get(0) * BM, col0 = blk.get(1) * BM;
        const double* A = a.rowData<double>(0);
        const double* B = b.rowData<double>(0);
        const std::size_t lda = a.leadingDim<double>(), ldb = b.leadingDim<double>();
        double accum[E][E];
#pragma unroll
        for (int i = 0; i < E; ++i)
#pragma unroll
            for (int j = 0; j < E; ++j)
                accum[i][j] = 0.0;
        for (std::size_t k0 = 0; k0 < n; k0 += BK) {
            for (int e = tid; e < BM * BK; e += T * T) { // A tile: BM rows x BK
                const int r = e / BK, kk = e % BK;
                const std::size_t gr = row0 + r, gk = k0 + kk;
                sa[r * (BK + 1) + kk] = gr < n && gk < n ? A[gr * lda + gk] : 0.0;
            }
            for (int e = tid; e < BK * BM; e += T * T) { // B tile: BK rows x BN
                const int kk = e / BM, col = e % BM;
                const std::size_t gk = k0 + kk, gc = col0 + col;
                sb[kk * (BM + 1) + col] = gk < n && gc < n ? B[gk * ldb + gc] : 0.0;
            }
            syncBlockThreads(acc);
#pragma unroll
            for (int kk = 0; kk < BK; ++kk) {
                double av[E], bv[E];
#pragma unroll
                for (int i = 0; i < E; ++i)
                    av[i] = sa[(ty + T * i) * (BK + 1) + kk];
#pragma unroll
                for (int j = 0; j < E; ++j)
                    bv[j] = sb[kk * (BM + 1) + tx + T * j];
#pragma unroll
                for (int i = 0; i < E; ++i)
#pragma unroll
                    for (int j = 0; j < E; ++j)
                        accum[i][j] = fma(av[i], bv[j], accum[i][j]);
            }
            syncBlockThreads(acc);
        }
#pragma unroll
        for (int i = 0; i < E; ++i) {
            const std::size_t r = row0 + ty + T * i;
            if (r >= n)
                continue;
            double* crow = c.rowData<double>(r);
#pragma unroll
            for (int j = 0; j < E; ++j) {
                const std::size_t col = col0 + tx + T * j;
                if (col < n)
                    crow[col] = alpha * accum[i][j] + beta * crow[col];
            }
        }
    }
};
KW_DEVICE_FUNCTOR(PaperHierarchicalGemm<4>)
KW_DEVICE_FUNCTOR(PaperHierarchicalGemm<8>)

template <int E>
double run_hierarchical(std::size_t n, Buffer& a, Buffer& b, Buffer& c)
{
    const WorkDiv wd(IndexVec((n + 16 * E - 1) / (16 * E), (n + 16 * E - 1) / (16 * E)), IndexVec(16, 16), IndexVec(E, E));
    executeTask(kBk, wd, PaperHierarchicalGemm<E>{}, n, 1.0, 0.0, view(a), view(b), view(c));
    std::vector<double> t;
    for (int r = 0; r < 3; ++r) {
        const auto t0 = std::chrono::steady_clock::now();
        executeTask(kBk, wd, PaperHierarchicalGemm<E>{}, n, 1.0, 0.0, view(a), view(b), view(c));
        t.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    }
    std::sort(t.begin(), t.end());
    return 2.0 * n * n * n / t[1] / 1e12;
}

TEST_CASE("paper's single-source hierarchical DGEMM functor: fraction of FP64 peak (PAPER.md:740-753)")
{
    const std::size_t n = 4096;
    Buffer ha(Device::host(), IndexVec(n, n), 8), hb(Device::host(), IndexVec(n, n), 8);
    std::mt19937_64 rng(4096);
    for (std::size_t r = 0; r < n; ++r)
        for (std::size_t col = 0; col < n; ++col) {
            ha.rowData<double>(r)[col] = static_cast<double>(rng() >> 11) * 0x1.0p-53 * 10.0;
            hb.rowData<double>(r)[col] = static_cast<double>(rng() >> 11) * 0x1.0p-53 * 10.0;
        }
    Buffer a(kGpu, IndexVec(n, n), 8), b(kGpu, IndexVec(n, n), 8), c(kGpu, IndexVec(n, n), 8), ref(kGpu, IndexVec(n, n), 8);
    {
        Queue q(kGpu, QueueFlavor::Sync);
        copyBuffer(q, a, ha, ha.extent());
        copyBuffer(q, b, hb, hb.extent());
        kw_memset(q.native(), ref.data(), 0, ref.storageBytes());
    }
    executeTask(kBk, kernels::gemmTiledWorkDiv(kBk, n, n, 128), kernels::GemmTiledKernel{},
                kernels::GemmArgs{n, n, n, 1.0, 0.0, &a, &b, &ref});
    const double peak = 37.22; // nominal FP64 (DMMA measured 37.16, DFMA 34.1: tools/probe/probe.cu)
    double best = 0.0;         // the paper picks the division per architecture: the best one counts
    for (int e : {4, 8}) {
        const double tf = e == 4 ? run_hierarchical<4>(n, a, b, c) : run_hierarchical<8>(n, a, b, c);
        // same product as the library's DGEMM within both kernels' (K+4)u bounds
        Buffer hc(Device::host(), IndexVec(n, n), 8), hr(Device::host(), IndexVec(n, n), 8);
        Queue q(kGpu, QueueFlavor::Sync);
        copyBuffer(q, hc, c, c.extent());
        copyBuffer(q, hr, ref, ref.extent());
        double worst = 0.0;
        for (std::size_t r = 0; r < n; r += 97)
            for (std::size_t col = 0; col < n; ++col) {
                const double x = hc.rowData<double>(r)[col], y = hr.rowData<double>(r)[col];
                worst = std::max(worst, std::fabs(x - y) / (std::fabs(y) * (2.0 * (n + 4)) * 0x1.0p-53));
            }
        std::printf("  single-source hierarchical DGEMM n=%zu, 16x16 threads x %dx%d elements: %.2f TFLOP/s = %.1f %% of "
                    "FP64 peak (paper: ~20 %%); max err / 2(K+4)u = %.3f\n",
                    n, e, e, tf, 100.0 * tf / peak, worst);
        CHECK(worst <= 1.0);
        best = std::max(best, tf / peak);
    }
    CHECK(best >= 0.20);
}

TEST_CASE("criterion 08 analogue: a generic functor runs within 1.5x of the native kernel (acceptance.cpp:546-587)")
{
    // The reference bounds library-kernel vs plain-loop medians by 1.5x. Here: the README AXPY
    // functor through the generic launcher vs the library's native AXPY kernel, n = 2^26 fp64
    // (1.6 GB of traffic per run, HBM-bound), medians of 9 synchronous executions.
    const std::size_t n = std::size_t{1} << 26;
    Buffer x(kGpu, IndexVec(n), 8), y(kGpu, IndexVec(n), 8);
    {
        Queue q(kGpu, QueueFlavor::Sync);
        kw_memset(q.native(), x.data(), 0, n * 8);
        kw_memset(q.native(), y.data(), 0, n * 8);
    }
    auto median_ms = [](auto&& run) {
        run();
        std::vector<double> t;
        for (int r = 0; r < 9; ++r) {
            const auto t0 = std::chrono::steady_clock::now();
            run();
            t.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
        }
        std::sort(t.begin(), t.end());
        return t[4];
    };
    const double native = median_ms([&] {
        executeTask(kBk, kernels::axpyWorkDiv(kBk, n, 512, 2), kernels::AxpyKernel{},
                    kernels::AxpyArgs{n, 0.5, &x, &y});
    });
    // Tuned division for this functor (it keeps the reference's per-thread contiguous chunk
    // [t*V, t*V+V), so lanes stride by V): 1024 threads x 2 elements. Measured (ms) for
    // tpb 128/256/512/1024 x V 1/2/3: 0.82/0.51/0.45, 0.50/0.35/0.34, 0.36/0.31/0.36,
    // 0.39/0.29/0.30 — native 0.25.
    const double functor = median_ms([&] {
        executeTask(kBk, divideForBackend(IndexVec(n), kBk, IndexVec(1024), IndexVec(2)), ScaleKernel{}, n, 0.5,
                    view(x), view(y));
    });
    std::printf("  axpy 2^26 f64: native %.3f ms, generic functor %.3f ms (%.2fx, bound 1.5x)\n", native, functor,
                functor / native);
    CHECK(functor <= 1.5 * native);
}

int main()
{
    if (deviceCount() == 0) {
        std::printf("no CUDA device\n");
        return 2;
    }
    return kwcheck::run();
}
