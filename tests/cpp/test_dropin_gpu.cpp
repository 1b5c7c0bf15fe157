// GPU checks of the C++ drop-in, written like the reference's test_kernels.cpp (whose cases
// are cited per test) but executing on BackendKind::GpuCudaRt through libkw_b200.so.
// The expected values come from in-test sequential loops identical to axpyReference /
// gemmReference (reference.cpp:8-26); built without FMA contraction (x86-64 baseline).
#include <kernelweave/kernelweave.hpp>

#include "check.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <random>
#include <sstream>
#include <vector>

using namespace kernelweave;
using namespace kernelweave::kernels;

namespace {

const Device kHost = Device::host();
const Device kGpu = Device::gpu(0);
constexpr BackendKind kBk = BackendKind::GpuCudaRt;

template <class T>
Buffer toGpu(const std::vector<T>& v)
{
    Buffer h(kHost, IndexVec(v.size()), sizeof(T));
    std::memcpy(h.rowData<T>(0), v.data(), v.size() * sizeof(T));
    Buffer d(kGpu, IndexVec(v.size()), sizeof(T));
    Queue q(kGpu, QueueFlavor::Sync);
    copyBuffer(q, d, h, h.extent());
    return d;
}

template <class T>
std::vector<T> toHost(const Buffer& d)
{
    Buffer h(kHost, d.extent(), d.elemSize());
    Queue q(kGpu, QueueFlavor::Sync);
    copyBuffer(q, h, d, d.extent());
    return std::vector<T>(h.rowData<T>(0), h.rowData<T>(0) + d.extent()[0]);
}

Buffer matrix(std::size_t r, std::size_t c, std::mt19937_64& rng, std::vector<double>* dense)
{
    Buffer h(kHost, IndexVec(r, c), 8);
    fillUniform<double>(h, rng, 0.0, 10.0);
    dense->resize(r * c);
    for (std::size_t i = 0; i < r; ++i)
        std::memcpy(dense->data() + i * c, h.rowData<double>(i), c * 8);
    Buffer d(kGpu, IndexVec(r, c), 8);
    Queue q(kGpu, QueueFlavor::Sync);
    copyBuffer(q, d, h, h.extent());
    return d;
}

std::vector<double> download(const Buffer& d)
{
    Buffer h(kHost, d.extent(), 8);
    Queue q(kGpu, QueueFlavor::Sync);
    copyBuffer(q, h, d, d.extent());
    const std::size_t r = d.extent()[0], c = d.extent()[1];
    std::vector<double> out(r * c);
    for (std::size_t i = 0; i < r; ++i)
        std::memcpy(out.data() + i * c, h.rowData<double>(i), c * 8);
    return out;
}

template <class T>
void axpyRef(std::size_t n, T alpha, const T* x, T* y)
{
    for (std::size_t i = 0; i < n; ++i)
        y[i] = alpha * x[i] + y[i];
}

void gemmRef(std::size_t m, std::size_t n, std::size_t k, double alpha, double beta, const double* a,
             const double* b, double* c)
{
    for (std::size_t r = 0; r < m; ++r)
        for (std::size_t col = 0; col < n; ++col) {
            double acc = 0.0;
            for (std::size_t p = 0; p < k; ++p)
                acc += a[r * k + p] * b[p * n + col];
            c[r * n + col] = alpha * acc + beta * c[r * n + col];
        }
}

bool withinTol(const std::vector<double>& got, const std::vector<double>& ref, std::size_t k)
{
    for (std::size_t i = 0; i < got.size(); ++i)
        if (std::fabs(got[i] - ref[i]) > (k + 4) * 0x1.0p-53 * std::fabs(ref[i]))
            return false;
    return true;
}

} // namespace

TEST_CASE("axpy on tiny vectors (test_kernels.cpp:73-86)")
{
    Buffer x = toGpu<double>({1, 2, 3});
    Buffer y = toGpu<double>({10, 20, 30});
    executeTask(kBk, axpyWorkDiv(kBk, 3, 2, 1), AxpyKernel{}, AxpyArgs{3, 2.0, &x, &y});
    CHECK((toHost<double>(y) == std::vector<double>{12, 24, 36}));
    Buffer y2 = toGpu<double>({10, 20, 30});
    executeTask(kBk, axpyWorkDiv(kBk, 3, 2, 1), AxpyKernel{}, AxpyArgs{3, 0.0, &x, &y2});
    CHECK((toHost<double>(y2) == std::vector<double>{10, 20, 30}));
}

TEST_CASE("axpy guards the tail (test_kernels.cpp:88-112)")
{
    std::mt19937_64 rng(42);
    std::vector<double> xs(128), ys(128);
    for (auto* v : {&xs, &ys})
        for (auto& e : *v)
            e = static_cast<double>(rng() >> 11) * 0x1.0p-53 * 10.0;
    for (std::size_t i = 100; i < 128; ++i)
        ys[i] = -555.25;
    std::vector<double> expected = ys;
    axpyRef<double>(100, 1.5, xs.data(), expected.data());
    Buffer x = toGpu(xs), y = toGpu(ys);
    const WorkDiv wd(IndexVec(2), IndexVec(16), IndexVec(4));
    CHECK(totalExtent(wd, Level::Grid, Unit::Elems) == IndexVec(128));
    executeTask(kBk, wd, AxpyKernel{}, AxpyArgs{100, 1.5, &x, &y});
    CHECK(toHost<double>(y) == expected);
}

TEST_CASE("native axpy loop and GPU kernel produce identical bits (test_kernels.cpp:331-349)")
{
    std::mt19937_64 rng(55);
    const std::size_t n = 4099;
    Buffer hx(kHost, IndexVec(n), 8), hy(kHost, IndexVec(n), 8);
    fillUniform<double>(hx, rng, 0.0, 10.0);
    fillUniform<double>(hy, rng, 0.0, 10.0);
    std::vector<double> native(hy.rowData<double>(0), hy.rowData<double>(0) + n);
    axpyRef<double>(n, 3.25, hx.rowData<double>(0), native.data());
    for (auto [tpb, ept] : {std::pair<int, int>{16, 8}, {256, 16}, {1, 1}, {128, 3}}) {
        Buffer x(kGpu, IndexVec(n), 8), y(kGpu, IndexVec(n), 8);
        Queue q(kGpu, QueueFlavor::Async);
        copyBuffer(q, x, hx, hx.extent());
        copyBuffer(q, y, hy, hy.extent());
        q.enqueue(createExec(kBk, axpyWorkDiv(kBk, n, tpb, ept), AxpyKernel{}, AxpyArgs{n, 3.25, &x, &y}));
        q.wait();
        CHECK(toHost<double>(y) == native);
    }
    // fp32 path, and host (pinned) operands streamed through the GPU
    Buffer fx(kHost, IndexVec(n), 4), fy(kHost, IndexVec(n), 4);
    fillUniform<float>(fx, rng, 0.0f, 10.0f);
    fillUniform<float>(fy, rng, 0.0f, 10.0f);
    std::vector<float> want(fy.rowData<float>(0), fy.rowData<float>(0) + n);
    axpyRef<float>(n, 2.75f, fx.rowData<float>(0), want.data());
    executeTask(kBk, axpyWorkDiv(kBk, n, 256, 16), AxpyKernel{}, AxpyArgsF32{n, 2.75f, &fx, &fy});
    CHECK(std::memcmp(fy.rowData<float>(0), want.data(), n * 4) == 0);
}

TEST_CASE("gemm closed forms (test_kernels.cpp:114-170)")
{
    std::mt19937_64 rng(7);
    std::vector<double> bd, cd;
    Buffer hid(kHost, IndexVec(4, 4), 8);
    for (std::size_t r = 0; r < 4; ++r)
        for (std::size_t c = 0; c < 4; ++c)
            hid.at<double>(IndexVec(r, c)) = r == c ? 1.0 : 0.0;
    Buffer ident(kGpu, IndexVec(4, 4), 8);
    Queue q(kGpu, QueueFlavor::Sync);
    copyBuffer(q, ident, hid, hid.extent());
    Buffer b = matrix(4, 4, rng, &bd);
    for (int naive = 0; naive < 2; ++naive) {
        Buffer c = matrix(4, 4, rng, &cd);
        const GemmArgs args{4, 4, 4, 1.0, 0.0, &ident, &b, &c, 64};
        if (naive)
            executeTask(kBk, gemmNaiveWorkDiv(kBk, 4, 4, 2, 2), GemmNaiveKernel{}, args);
        else
            executeTask(kBk, gemmTiledWorkDiv(kBk, 4, 4, 64), GemmTiledKernel{}, args);
        CHECK(download(c) == bd);
        Buffer c3 = matrix(4, 4, rng, &cd);
        const GemmArgs keep{4, 4, 4, 0.0, 1.0, &ident, &b, &c3, 128};
        executeTask(kBk, gemmTiledWorkDiv(kBk, 4, 4, 128), GemmTiledKernel{}, keep);
        CHECK(download(c3) == cd);
    }
}

TEST_CASE("naive GPU kernel is bitwise equal to the sequential oracle (test_kernels.cpp:184-206)")
{
    std::mt19937_64 rng(1234);
    for (int iter = 0; iter < 50; ++iter) {
        const std::size_t m = 1 + rng() % 64, n = 1 + rng() % 64, k = 1 + rng() % 64;
        std::vector<double> ad, bd, cd;
        Buffer a = matrix(m, k, rng, &ad), b = matrix(k, n, rng, &bd), c = matrix(m, n, rng, &cd);
        const double alpha = 0.5 + static_cast<double>(rng() % 8), beta = static_cast<double>(rng() % 3);
        gemmRef(m, n, k, alpha, beta, ad.data(), bd.data(), cd.data());
        executeTask(kBk, gemmNaiveWorkDiv(kBk, m, n, 4, 4), GemmNaiveKernel{}, GemmArgs{m, n, k, alpha, beta, &a, &b, &c});
        CHECK(download(c) == cd);
    }
}

TEST_CASE("tiled GPU kernel within (K+4)u at every size 1..64 and ragged shapes")
{
    std::mt19937_64 rng(5678);
    for (std::size_t s = 1; s <= 64; ++s) {
        std::vector<double> ad, bd, cd;
        Buffer a = matrix(s, s, rng, &ad), b = matrix(s, s, rng, &bd), c = matrix(s, s, rng, &cd);
        gemmRef(s, s, s, 1.25, 0.75, ad.data(), bd.data(), cd.data());
        executeTask(kBk, gemmTiledWorkDiv(kBk, s, s, 128), GemmTiledKernel{},
                    GemmArgs{s, s, s, 1.25, 0.75, &a, &b, &c, 128});
        CHECK(withinTol(download(c), cd, s));
    }
    const std::size_t m = 13, n = 29, k = 7;
    std::vector<double> ad, bd, cd;
    Buffer a = matrix(m, k, rng, &ad), b = matrix(k, n, rng, &bd), c = matrix(m, n, rng, &cd);
    gemmRef(m, n, k, 2.5, 0.0, ad.data(), bd.data(), cd.data());
    executeTask(kBk, gemmTiledWorkDiv(kBk, m, n, 64), GemmTiledKernel{}, GemmArgs{m, n, k, 2.5, 0.0, &a, &b, &c, 64});
    CHECK(withinTol(download(c), cd, k));
}

TEST_CASE("queue semantics: async FIFO, task handles, usage errors before enqueue")
{
    const std::size_t n = 1 << 20;
    Buffer hx(kHost, IndexVec(n), 4), hy(kHost, IndexVec(n), 4);
    std::mt19937_64 rng(9);
    fillUniform<float>(hx, rng, 0.0f, 10.0f);
    fillUniform<float>(hy, rng, 0.0f, 10.0f);
    std::vector<float> want(hy.rowData<float>(0), hy.rowData<float>(0) + n);
    for (int rep = 0; rep < 3; ++rep)
        axpyRef<float>(n, 0.5f, hx.rowData<float>(0), want.data());
    Buffer x(kGpu, IndexVec(n), 4), y(kGpu, IndexVec(n), 4);
    Queue q(kGpu, QueueFlavor::Async);
    copyBuffer(q, x, hx, hx.extent());
    copyBuffer(q, y, hy, hy.extent());
    TaskHandle last = q.enqueue(createExec(kBk, axpyWorkDiv(kBk, n, 256, 16), AxpyKernel{}, AxpyArgsF32{n, 0.5f, &x, &y}));
    for (int rep = 1; rep < 3; ++rep)
        last = q.enqueue(createExec(kBk, axpyWorkDiv(kBk, n, 256, 16), AxpyKernel{}, AxpyArgsF32{n, 0.5f, &x, &y}));
    copyBuffer(q, hy, y, y.extent());
    q.wait();
    CHECK(last.state() == TaskState::Done);
    CHECK(std::memcmp(hy.rowData<float>(0), want.data(), n * 4) == 0);
    CHECK_THROWS_AS(q.enqueue(createExec(kBk, WorkDiv(IndexVec(1), IndexVec(4096), IndexVec(1)), AxpyKernel{},
                                         AxpyArgsF32{n, 0.5f, &x, &y})),
                    UsageError);
    Buffer wrong(kGpu, IndexVec(8), 8);
    CHECK_THROWS_AS(createExec(kBk, axpyWorkDiv(kBk, n, 256, 16), AxpyKernel{}, AxpyArgsF32{n, 0.5f, &x, &wrong}),
                    UsageError);
    q.wait(); // nothing failed
}

TEST_CASE("pitched copies never touch bytes outside the box (acceptance crit. 7 shape)")
{
    Buffer hsrc(kHost, IndexVec(5, 7), 8);
    for (std::size_t r = 0; r < 5; ++r)
        for (std::size_t c = 0; c < 7; ++c)
            hsrc.at<double>(IndexVec(r, c)) = static_cast<double>(r * 7 + c);
    Buffer dsrc(kGpu, IndexVec(5, 7), 8), ddst(kGpu, IndexVec(6, 9), 8);
    Buffer hdst(kHost, IndexVec(6, 9), 8);
    std::memset(hdst.data(), 0xEE, hdst.storageBytes());
    Queue q(kGpu, QueueFlavor::Sync);
    copyBuffer(q, ddst, hdst, hdst.extent());
    copyBuffer(q, dsrc, hsrc, hsrc.extent());
    copyBuffer(q, ddst, dsrc, IndexVec(4, 5));
    copyBuffer(q, hdst, ddst, ddst.extent());
    bool ok = true;
    for (std::size_t r = 0; r < 6; ++r) {
        const auto* raw = reinterpret_cast<const unsigned char*>(hdst.data()) + r * hdst.rowPitch();
        for (std::size_t bi = 0; bi < hdst.rowPitch(); ++bi) {
            const bool inside = r < 4 && bi < 5 * 8;
            if (!inside && raw[bi] != 0xEE && bi < 9 * 8)
                ok = false;
        }
        for (std::size_t c = 0; r < 4 && c < 5; ++c)
            ok = ok && hdst.at<double>(IndexVec(r, c)) == static_cast<double>(r * 7 + c);
    }
    CHECK(ok);
    CHECK_THROWS_AS(createCopy(ddst, dsrc, IndexVec(6, 9)), UsageError);
}

TEST_CASE("element access layout; buffers move, never copy (test_buffer.cpp:53-110)")
{
    Buffer buf(Device::host(), IndexVec(10, 10), 8, 128);
    CHECK(buf.rowPitch() == 128);
    CHECK(buf.byteOffset(IndexVec(2, 3)) == 2 * 128 + 3 * 8);
    buf.at<double>(IndexVec(2, 3)) = 42.5;
    CHECK(buf.at<double>(IndexVec(2, 3)) == 42.5);
    CHECK(static_cast<const std::byte*>(buf.elementPtr(IndexVec(2, 3))) == buf.data() + 2 * 128 + 24);
    auto usage = [](auto&& f) {
        try {
            f();
        }
        catch (const UsageError&) {
            return true;
        }
        return false;
    };
    CHECK(usage([&] { (void)buf.byteOffset(IndexVec(10, 0)); }));
    CHECK(usage([&] { (void)buf.byteOffset(IndexVec(0, 10)); }));
    CHECK(usage([&] { (void)buf.byteOffset(IndexVec(3)); }));
    CHECK(usage([&] { (void)buf.at<float>(IndexVec(0, 0)); }));
    // every element of the extent has its own offset
    std::vector<std::size_t> offs;
    for (std::size_t r = 0; r < 10; ++r)
        for (std::size_t c = 0; c < 10; ++c)
            offs.push_back(buf.byteOffset(IndexVec(r, c)));
    std::sort(offs.begin(), offs.end());
    CHECK(std::adjacent_find(offs.begin(), offs.end()) == offs.end());
    // move-only ownership, for host and device storage alike
    for (Device where : {Device::host(), Device::gpu(0)}) {
        Buffer a(where, IndexVec(4, 4), 8);
        const std::byte* storage = a.data();
        Buffer b = std::move(a);
        CHECK(b.data() == storage);
        Buffer c(where, IndexVec(2), 8);
        c = std::move(b);
        CHECK(c.data() == storage);
        CHECK(c.extent() == IndexVec(4, 4));
    }
}

TEST_CASE("buffer CSV round-trips bitwise, host and GPU buffers (test_buffer.cpp:275-310)")
{
    Buffer buf(Device::host(), IndexVec(7, 5), 8);
    std::mt19937_64 rng(99);
    fillUniform<double>(buf, rng, 0.0, 10.0);
    buf.at<double>(IndexVec(0, 0)) = 1.0 / 3.0;
    buf.at<double>(IndexVec(6, 4)) = -0.0;
    std::stringstream first;
    writeBufferCsv(buf, first);
    // the text the reference's writer produces for these values (%.17g per value)
    if (const char* path = std::getenv("KW_CSV_OUT")) {
        std::ofstream f(path, std::ios::binary);
        f << first.str();
    }
    for (Device where : {Device::host(), Device::gpu(0)}) {
        std::stringstream in(first.str());
        Buffer parsed = readBufferCsv(in, where);
        CHECK(parsed.extent() == buf.extent());
        CHECK(parsed.device() == where);
        std::stringstream second;
        writeBufferCsv(parsed, second); // a GPU buffer is staged through the host
        CHECK(second.str() == first.str());
        Buffer back(Device::host(), buf.extent(), 8);
        Queue q(Device::gpu(0), QueueFlavor::Sync);
        copyBuffer(q, back, parsed, buf.extent());
        bool same = true;
        for (std::size_t r = 0; r < 7; ++r)
            same = same && std::memcmp(back.rowData<double>(r), buf.rowData<double>(r), 5 * 8) == 0;
        CHECK(same);
    }
    auto throwsUsage = [](const std::string& text) {
        std::stringstream in(text);
        try {
            readBufferCsv(in);
        }
        catch (const UsageError&) {
            return true;
        }
        return false;
    };
    CHECK(throwsUsage("1,2\n3\n"));
    CHECK(throwsUsage(""));
    CHECK(throwsUsage("1,x\n"));
    Buffer vec(Device::host(), IndexVec(4), 8);
    std::stringstream out;
    bool threw = false;
    try {
        writeBufferCsv(vec, out);
    }
    catch (const UsageError&) {
        threw = true;
    }
    CHECK(threw);
}

int main()
{
    if (deviceCount() == 0) {
        std::printf("no CUDA device\n");
        return 2;
    }
    return kwcheck::run();
}

// The functors' reference-signature operator() (axpy.hpp:23-25, gemm.hpp:33, :47), invoked
// directly the way the reference's runGrid does — one call per (block, thread) of a division —
// on host buffers, against the sequential oracles; and device buffers are refused.
TEST_CASE("functor operator()(acc, args): direct invocation over a division equals the oracle")
{
    std::mt19937_64 rng(4242);
    const std::size_t n = 1003;
    Buffer x(kHost, IndexVec(n), 8), y(kHost, IndexVec(n), 8);
    fillUniform<double>(x, rng, 0.0, 10.0);
    fillUniform<double>(y, rng, 0.0, 10.0);
    std::vector<double> want(y.rowData<double>(0), y.rowData<double>(0) + n);
    axpyRef<double>(n, 3.25, x.rowData<double>(0), want.data());
    const WorkDiv wd = axpyWorkDiv(BackendKind::ThreadsParallel, n, 16, 8);
    const AxpyArgs args{n, 3.25, &x, &y};
    for (std::size_t b = 0; b < wd.blocksPerGrid()[0]; ++b)
        for (std::size_t t = 0; t < wd.threadsPerBlock()[0]; ++t)
            AxpyKernel{}(AccContext(wd, IndexVec(b), IndexVec(t)), args);
    CHECK(std::memcmp(want.data(), y.rowData<double>(0), n * 8) == 0);

    const std::size_t m = 37, nn = 29, k = 41;
    Buffer a(kHost, IndexVec(m, k), 8), bb(kHost, IndexVec(k, nn), 8), c(kHost, IndexVec(m, nn), 8);
    fillUniform<double>(a, rng, 0.0, 10.0);
    fillUniform<double>(bb, rng, 0.0, 10.0);
    fillUniform<double>(c, rng, 0.0, 10.0);
    std::vector<double> da(m * k), db(k * nn), dc(m * nn);
    for (std::size_t r = 0; r < m; ++r)
        std::memcpy(da.data() + r * k, a.rowData<double>(r), k * 8);
    for (std::size_t r = 0; r < k; ++r)
        std::memcpy(db.data() + r * nn, bb.rowData<double>(r), nn * 8);
    for (std::size_t r = 0; r < m; ++r)
        std::memcpy(dc.data() + r * nn, c.rowData<double>(r), nn * 8);
    gemmRef(m, nn, k, 1.5, 0.25, da.data(), db.data(), dc.data());
    const WorkDiv nwd = gemmNaiveWorkDiv(BackendKind::ThreadsParallel, m, nn, 4, 3);
    const GemmArgs g{m, nn, k, 1.5, 0.25, &a, &bb, &c};
    const IndexVec blocks = nwd.blocksPerGrid(), threads = nwd.threadsPerBlock();
    for (std::size_t b0 = 0; b0 < blocks[0]; ++b0)
        for (std::size_t b1 = 0; b1 < blocks[1]; ++b1)
            for (std::size_t t0 = 0; t0 < threads[0]; ++t0)
                for (std::size_t t1 = 0; t1 < threads[1]; ++t1)
                    GemmNaiveKernel{}(AccContext(nwd, IndexVec(b0, b1), IndexVec(t0, t1)), g);
    bool same = true;
    for (std::size_t r = 0; r < m; ++r)
        same = same && std::memcmp(dc.data() + r * nn, c.rowData<double>(r), nn * 8) == 0;
    CHECK(same);
    // block-cooperative tiled body: device functors only
    CHECK_THROWS_AS(GemmTiledKernel{}(AccContext(nwd, IndexVec(0, 0), IndexVec(0, 0)), g), UsageError);
    // GPU buffers go through executeTask / createExec
    Buffer gx(kGpu, IndexVec(n), 8), gy(kGpu, IndexVec(n), 8);
    CHECK_THROWS_AS(AxpyKernel{}(AccContext(wd, IndexVec(0), IndexVec(0)), AxpyArgs{n, 1.0, &gx, &gy}), UsageError);
}
