// kwbench for the B200 build — the reference's benchmark harness contract (tools/bench/main.cpp,
// runner.cpp:238-355, records.cpp) on the drop-in API.
//
//   kwbench --kernel axpy|gemm-naive|gemm-tiled [--backend gpu|native|all] [--sizes a,b,..]
//           [--reps N>=3] [--seed S] [--tile T] [--tpb B] [--ept V] [--dtype f64|f32] [--verify]
//           [--csv PATH] [--baseline gpu|native] [--pessimize]
//
// Back-ends: "gpu" = the library's kernels through createExec/Queue; "native" = plain CUDA kernels
// launched directly on the raw device pointers, without the library's API — the GPU counterpart
// of the reference's native loops (runner.cpp:160-171; the zero-overhead analogue of acceptance
// criterion 08): a grid-stride AXPY and a one-thread-per-element GEMM with the reference's exact
// arithmetic (bitwise equal to axpyReference / gemmReference). --baseline prints every median
// relative to that back-end (benchmarked if not selected, relativeReport runner.cpp:303-328);
// --pessimize adds the degraded division and its slowdown summary (runner.cpp:330-355).
//
// Per point (runner.cpp:252-281): seed-deterministic uniform [0,10) inputs drawn exactly like
// Workload (seed_seq{seed, n, fnv1a(kernel)}, alpha, beta, fillUniform — runner.cpp:56-85), one
// untimed warm-up, then each rep restores the output (untimed device copy), times exactly the
// enqueue + wait with the steady clock, and with --verify compares against the sequential
// reference loop: bitwise for axpy and gemm-naive, |dC| <= (K+4)*2^-53*|C| for gemm-tiled.
// CSV columns are the reference's: kernel,backend,n,b,v,tile,rep,seconds,gflops,verified
// (%.17g, records.cpp:17-42). Exit codes: 0 ok, 1 verification failure, 2 usage error.
#include <kernelweave/kernelweave.hpp>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

using namespace kernelweave;
using namespace kernelweave::kernels;

namespace {

using Clock = std::chrono::steady_clock;

// ---- the "native" back-end: plain CUDA, no kernelweave API ---------------------------------
__device__ __forceinline__ float native_axpy1(float a, float x, float y) { return __fadd_rn(__fmul_rn(a, x), y); }
__device__ __forceinline__ double native_axpy1(double a, double x, double y) { return __dadd_rn(__dmul_rn(a, x), y); }

template <class T>
__global__ void native_axpy(std::size_t n, T a, const T* __restrict__ x, T* __restrict__ y)
{
    const std::size_t stride = static_cast<std::size_t>(gridDim.x) * blockDim.x;
    for (std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        y[i] = native_axpy1(a, x[i], y[i]);
}

// C = alpha*A*B + beta*C, one thread per element, ascending p, separately rounded (gemmReference)
__global__ void native_gemm(std::size_t n, double alpha, double beta, const double* __restrict__ A, std::size_t lda,
                            const double* __restrict__ B, std::size_t ldb, double* __restrict__ C, std::size_t ldc)
{
    const std::size_t c = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const std::size_t r = static_cast<std::size_t>(blockIdx.y) * blockDim.y + threadIdx.y;
    if (r >= n || c >= n)
        return;
    double acc = 0.0;
    for (std::size_t p = 0; p < n; ++p)
        acc = __dadd_rn(acc, __dmul_rn(A[r * lda + p], B[p * ldb + c]));
    C[r * ldc + c] = __dadd_rn(__dmul_rn(alpha, acc), __dmul_rn(beta, C[r * ldc + c]));
}

cudaStream_t streamOf(Queue& q)
{
    void* s = nullptr;
    detail::check(kw_queue_stream(q.native(), &s));
    return static_cast<cudaStream_t>(s);
}

// KWBENCH_INJECT_FAULT (runner.cpp:28-32): corrupt one output byte after every timed run so the
// verification-failure path (exit code 1) can be exercised end to end.
bool injectFault()
{
    const char* raw = std::getenv("KWBENCH_INJECT_FAULT");
    return raw != nullptr && *raw != '\0';
}

struct Config {
    std::string kernel = "axpy";
    std::string backend = "gpu";
    std::vector<std::size_t> sizes = {256};
    int reps = 5;
    std::uint64_t seed = 42;
    std::size_t tile = 128, tpb = 512, ept = 4;
    bool tpb_set = false, ept_set = false; // gemm-naive has its own tuned default division
    bool verify = false, pessimize = false, f32 = false;
    std::string csv, baseline;
    std::vector<std::string> backends; // resolved from --backend (+ the baseline if missing)
};

struct Record {
    std::string kernel, backend;
    std::size_t n, b, v, tile;
    int rep;
    double seconds, gflops;
    bool verified;
};

std::string fmt(double v)
{
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
}

std::uint64_t kernelTag(const std::string& k)
{
    std::uint64_t h = 1469598103934665603ull;
    for (char ch : k) {
        h ^= static_cast<unsigned char>(ch);
        h *= 1099511628211ull;
    }
    return h;
}

double flopCount(const std::string& k, std::size_t n)
{
    const double d = static_cast<double>(n);
    return k == "axpy" ? 2.0 * d : 2.0 * d * d * d + 3.0 * d * d;
}

std::vector<std::size_t> parseSizes(const std::string& s)
{
    std::vector<std::size_t> out;
    std::stringstream ss(s);
    std::string tok;
    while (std::getline(ss, tok, ',')) {
        char* end = nullptr;
        const unsigned long long v = std::strtoull(tok.c_str(), &end, 10);
        if (end == tok.c_str() || *end)
            throw UsageError("malformed size '" + tok + "'");
        out.push_back(v);
    }
    return out;
}

Config parse(int argc, char** argv)
{
    Config c;
    for (int i = 1; i < argc; ++i) {
        const std::string a = argv[i];
        auto val = [&]() -> std::string {
            if (i + 1 >= argc)
                throw UsageError("missing value for " + a);
            return argv[++i];
        };
        if (a == "--kernel")
            c.kernel = val();
        else if (a == "--backend")
            c.backend = val();
        else if (a == "--sizes")
            c.sizes = parseSizes(val());
        else if (a == "--reps")
            c.reps = std::atoi(val().c_str());
        else if (a == "--seed")
            c.seed = std::strtoull(val().c_str(), nullptr, 10);
        else if (a == "--tile")
            c.tile = std::strtoull(val().c_str(), nullptr, 10);
        else if (a == "--tpb") {
            c.tpb = std::strtoull(val().c_str(), nullptr, 10);
            c.tpb_set = true;
        }
        else if (a == "--ept") {
            c.ept = std::strtoull(val().c_str(), nullptr, 10);
            c.ept_set = true;
        }
        else if (a == "--dtype") {
            const std::string d = val();
            if (d != "f32" && d != "f64")
                throw UsageError("--dtype must be f32 or f64");
            c.f32 = d == "f32";
        }
        else if (a == "--verify")
            c.verify = true;
        else if (a == "--pessimize")
            c.pessimize = true;
        else if (a == "--csv")
            c.csv = val();
        else if (a == "--baseline")
            c.baseline = val();
        else
            throw UsageError("unknown option " + a);
    }
    // runner.cpp:199-218
    if (c.kernel != "axpy" && c.kernel != "gemm-naive" && c.kernel != "gemm-tiled")
        throw UsageError("unknown kernel '" + c.kernel + "' (expected axpy, gemm-naive or gemm-tiled)");
    if (c.backend == "all")
        c.backends = {"gpu", "native"};
    else if (c.backend == "gpu" || c.backend == "native")
        c.backends = {c.backend};
    else
        throw UsageError("backend '" + c.backend + "' does not exist in the B200 build (gpu, native or all)");
    if (!c.baseline.empty()) {
        if (c.baseline != "gpu" && c.baseline != "native")
            throw UsageError("baseline '" + c.baseline + "' is not a back-end (gpu or native)");
        if (std::find(c.backends.begin(), c.backends.end(), c.baseline) == c.backends.end())
            c.backends.push_back(c.baseline); // benchmarked when missing (runner.cpp:238-251)
    }
    if (c.reps < 3)
        throw UsageError("reps must be at least 3");
    if (c.sizes.empty())
        throw UsageError("at least one size is required");
    for (std::size_t n : c.sizes)
        if (n == 0)
            throw UsageError("sizes must be at least 1");
    // A tuned division per kernel, as acceptance.cpp:567-579 picks one for its gemm instances:
    // gemm-naive defaults to 16 threads x 16 elements (a 16 x 16 output block per CUDA block, one
    // output per CUDA thread); axpy keeps 512 x 4.
    if (c.kernel == "gemm-naive") {
        if (!c.tpb_set)
            c.tpb = 16;
        if (!c.ept_set)
            c.ept = 16;
    }
    if (c.tile == 0 || c.tpb == 0 || c.ept == 0)
        throw UsageError("tile, tpb and ept must be at least 1");
    if (c.pessimize && c.kernel == "axpy")
        throw UsageError("--pessimize applies to the gemm kernels only");
    if (c.f32 && c.kernel != "axpy")
        throw UsageError("--dtype f32 applies to axpy only (the gemm kernels are fp64)");
    return c;
}

template <class T>
Buffer hostFilled(const IndexVec& ext, std::mt19937_64& rng)
{
    Buffer b(Device::host(), ext, sizeof(T));
    fillUniform<T>(b, rng, T(0), T(10));
    return b;
}

Buffer toDevice(Queue& q, const Buffer& h)
{
    Buffer d(Device::gpu(0), h.extent(), h.elemSize());
    copyBuffer(q, d, h, h.extent());
    return d;
}

template <class T>
bool sameBits(const Buffer& a, const Buffer& b)
{
    for (std::size_t r = 0; r < a.rowCount(); ++r)
        if (std::memcmp(a.rowData<T>(r), b.rowData<T>(r), a.rowBytes()) != 0)
            return false;
    return true;
}

struct Point {
    std::vector<Record> records;
    bool failed = false;
};

template <class T>
Point runAxpy(const Config& c, std::size_t n, Queue& q, const std::string& backend)
{
    const bool native = backend == "native";
    std::seed_seq seq{c.seed, static_cast<std::uint64_t>(n), kernelTag("axpy")};
    std::mt19937_64 rng(seq);
    const double alpha = static_cast<double>(rng() >> 11) * 0x1.0p-53 * 10.0;
    (void)rng(); // beta, drawn and unused (runner.cpp:64-65)
    Buffer hx = hostFilled<T>(IndexVec(n), rng), hy = hostFilled<T>(IndexVec(n), rng);
    Buffer x = toDevice(q, hx), y0 = toDevice(q, hy), y = toDevice(q, hy);
    q.wait();
    Buffer ref(Device::host(), IndexVec(n), sizeof(T)), out(Device::host(), IndexVec(n), sizeof(T));
    if (c.verify) {
        std::memcpy(ref.data(), hy.data(), n * sizeof(T));
        T* r = ref.rowData<T>(0);
        const T* xs = hx.rowData<T>(0);
        const T a = static_cast<T>(alpha);
        for (std::size_t i = 0; i < n; ++i) // axpyReference (reference.cpp:8-12)
            r[i] = a * xs[i] + r[i];
    }
    const WorkDiv wd = axpyWorkDiv(BackendKind::GpuCudaRt, n, c.tpb, c.ept);
    Point pt;
    for (int rep = -1; rep < c.reps; ++rep) {
        copyBuffer(q, y, y0, y0.extent()); // restoreOutput (runner.cpp:97-100), untimed
        q.wait();
        ExecTask task = createExec(BackendKind::GpuCudaRt, wd, AxpyKernel{},
                                   AxpyArgsT<T>{n, static_cast<T>(alpha), &x, &y});
        const unsigned grid = static_cast<unsigned>(std::min<std::size_t>((n + 255) / 256, 148 * 8));
        const auto t0 = Clock::now();
        if (native) {
            native_axpy<T><<<grid, 256, 0, streamOf(q)>>>(n, static_cast<T>(alpha), x.rowData<T>(0), y.rowData<T>(0));
            if (cudaGetLastError() != cudaSuccess)
                throw std::runtime_error("native axpy launch failed");
        }
        else {
            q.enqueue(std::move(task));
        }
        q.wait();
        const double s = std::chrono::duration<double>(Clock::now() - t0).count();
        if (rep < 0)
            continue; // warm-up, discarded
        bool ok = true;
        if (c.verify) {
            copyBuffer(q, out, y, y.extent());
            q.wait();
            if (injectFault())
                out.data()[0] ^= std::byte{0x01};
            ok = sameBits<T>(out, ref);
        }
        pt.failed |= !ok;
        pt.records.push_back({"axpy", backend, n, native ? 256 : wd.threadsPerBlock().product(),
                              native ? 1 : wd.elementsPerThread().product(), 0, rep, s,
                              flopCount("axpy", n) / s / 1e9, ok});
    }
    return pt;
}

Point runGemm(const Config& c, std::size_t n, Queue& q, bool pessimized, const std::string& backend)
{
    const bool native = backend == "native";
    std::seed_seq seq{c.seed, static_cast<std::uint64_t>(n), kernelTag(c.kernel)};
    std::mt19937_64 rng(seq);
    const double alpha = static_cast<double>(rng() >> 11) * 0x1.0p-53 * 10.0;
    const double beta = static_cast<double>(rng() >> 11) * 0x1.0p-53 * 10.0;
    Buffer ha = hostFilled<double>(IndexVec(n, n), rng), hb = hostFilled<double>(IndexVec(n, n), rng),
           hc = hostFilled<double>(IndexVec(n, n), rng);
    Buffer a = toDevice(q, ha), b = toDevice(q, hb), c0 = toDevice(q, hc), cc = toDevice(q, hc);
    q.wait();
    Buffer ref(Device::host(), IndexVec(n, n), 8), out(Device::host(), IndexVec(n, n), 8);
    if (c.verify) { // gemmReference (reference.cpp:14-26), i-k-j order: same per-element sequence
        std::vector<double> acc(n);
        for (std::size_t r = 0; r < n; ++r) {
            std::fill(acc.begin(), acc.end(), 0.0);
            for (std::size_t p = 0; p < n; ++p) {
                const double av = ha.rowData<double>(r)[p];
                const double* brow = hb.rowData<double>(p);
                for (std::size_t col = 0; col < n; ++col)
                    acc[col] += av * brow[col];
            }
            for (std::size_t col = 0; col < n; ++col)
                ref.rowData<double>(r)[col] = alpha * acc[col] + beta * hc.rowData<double>(r)[col];
        }
    }
    // --pessimize (runner.cpp:148-153, acceptance crit. 10): gemm-naive degrades to one thread
    // owning the whole output; gemm-tiled degrades to "tile = 1" — each thread one output
    // element, no shared-memory reuse (the untiled kernel) — recorded with tile 1 like the
    // reference's degraded rows.
    const bool tiled = c.kernel == "gemm-tiled" && !pessimized && !native;
    const std::size_t tile = pessimized ? 1 : c.tile;
    const WorkDiv wd = tiled ? gemmTiledWorkDiv(BackendKind::GpuCudaRt, n, n, tile)
                       : !pessimized ? gemmNaiveWorkDiv(BackendKind::GpuCudaRt, n, n, c.tpb, c.ept)
                       : c.kernel == "gemm-tiled" ? gemmNaiveWorkDiv(BackendKind::GpuCudaRt, n, n, 16, 1)
                                                  : WorkDiv(IndexVec(1, 1), IndexVec(1, 1), IndexVec(n, n));
    const GemmArgs args{n, n, n, alpha, beta, &a, &b, &cc, tile};
    Point pt;
    for (int rep = -1; rep < c.reps; ++rep) {
        copyBuffer(q, cc, c0, c0.extent());
        q.wait();
        ExecTask task = tiled ? createExec(BackendKind::GpuCudaRt, wd, GemmTiledKernel{}, args)
                              : createExec(BackendKind::GpuCudaRt, wd, GemmNaiveKernel{}, args);
        const auto t0 = Clock::now();
        if (native) {
            native_gemm<<<dim3(static_cast<unsigned>((n + 15) / 16), static_cast<unsigned>((n + 15) / 16)), dim3(16, 16), 0,
                          streamOf(q)>>>(n, alpha, beta, a.rowData<double>(0), a.leadingDim<double>(),
                                         b.rowData<double>(0), b.leadingDim<double>(), cc.rowData<double>(0),
                                         cc.leadingDim<double>());
            if (cudaGetLastError() != cudaSuccess)
                throw std::runtime_error("native gemm launch failed");
        }
        else {
            q.enqueue(std::move(task));
        }
        q.wait();
        const double s = std::chrono::duration<double>(Clock::now() - t0).count();
        if (rep < 0)
            continue;
        bool ok = true;
        if (c.verify) {
            copyBuffer(q, out, cc, cc.extent());
            q.wait();
            if (injectFault())
                out.data()[0] ^= std::byte{0x40};
            if (tiled) {
                for (std::size_t r = 0; r < n && ok; ++r)
                    for (std::size_t col = 0; col < n; ++col) {
                        const double g = out.rowData<double>(r)[col], w = ref.rowData<double>(r)[col];
                        if (std::fabs(g - w) > (n + 4) * 0x1.0p-53 * std::fabs(w)) {
                            ok = false;
                            break;
                        }
                    }
            }
            else {
                ok = sameBits<double>(out, ref);
            }
        }
        pt.failed |= !ok;
        pt.records.push_back({c.kernel, backend, n, native ? 256 : wd.threadsPerBlock().product(),
                              native ? 1 : wd.elementsPerThread().product(),
                              c.kernel == "gemm-tiled" && !native ? tile : 0, rep, s, flopCount(c.kernel, n) / s / 1e9,
                              ok});
    }
    return pt;
}

double median(std::vector<double> v)
{
    std::sort(v.begin(), v.end());
    const std::size_t m = v.size() / 2;
    return v.size() % 2 ? v[m] : (v[m - 1] + v[m]) / 2.0;
}

} // namespace

int main(int argc, char** argv)
{
    Config cfg;
    try {
        cfg = parse(argc, argv);
    }
    catch (const UsageError& e) {
        std::fprintf(stderr, "kwbench: %s\n", e.what());
        return 2;
    }
    if (deviceCount() == 0) {
        std::fprintf(stderr, "kwbench: no CUDA device\n");
        return 2;
    }
    std::vector<Record> all;
    bool failed = false;
    try {
        Queue q(Device::gpu(0), QueueFlavor::Sync);
        for (std::size_t n : cfg.sizes) {
            std::vector<Point> pts;
            for (const std::string& be : cfg.backends) {
                if (cfg.kernel == "axpy")
                    pts.push_back(cfg.f32 ? runAxpy<float>(cfg, n, q, be) : runAxpy<double>(cfg, n, q, be));
                else {
                    pts.push_back(runGemm(cfg, n, q, false, be));
                    if (cfg.pessimize && be == "gpu") // a division of the library's kernels
                        pts.push_back(runGemm(cfg, n, q, true, be));
                }
            }
            for (auto& p : pts) {
                failed |= p.failed;
                std::vector<double> secs;
                for (auto& r : p.records)
                    secs.push_back(r.seconds);
                const double med = median(secs);
                const Record& r0 = p.records.front();
                const double bytes = cfg.kernel == "axpy" ? 3.0 * n * (cfg.f32 ? 4 : 8) : 0.0;
                std::printf("%-10s %-6s n=%-9zu b=%-5zu v=%-7zu tile=%-4zu median %.6g s  %.4g GFLOP/s%s%s\n",
                            r0.kernel.c_str(), r0.backend.c_str(), n, r0.b, r0.v, r0.tile, med,
                            flopCount(cfg.kernel, n) / med / 1e9,
                            bytes > 0 ? ("  " + fmt(bytes / med / 1e9) + " GB/s").c_str() : "",
                            cfg.verify ? (p.failed ? "  VERIFY FAILED" : "  verified") : "");
                all.insert(all.end(), p.records.begin(), p.records.end());
            }
        }
    }
    catch (const std::exception& e) {
        std::fprintf(stderr, "kwbench: %s\n", e.what());
        return 2;
    }
    // pessimizeSummary (runner.cpp:330-355): degraded vs tuned division, per point
    auto medianOf = [&](const std::string& be, std::size_t n, int pess) {
        std::vector<double> v;
        for (const auto& r : all) {
            const bool degraded = cfg.kernel == "gemm-tiled" ? (r.tile == 1 && cfg.tile != 1) : (r.v == r.n * r.n);
            if (r.backend == be && r.n == n && (pess < 0 || degraded == (pess == 1)))
                v.push_back(r.seconds);
        }
        return v.empty() ? 0.0 : median(v);
    };
    if (cfg.pessimize) {
        std::printf("\npessimized division slowdown (median vs tuned division):\n");
        for (std::size_t n : cfg.sizes) {
            const double tuned = medianOf("gpu", n, 0), bad = medianOf("gpu", n, 1);
            if (tuned > 0.0 && bad > 0.0)
                std::printf("  %s gpu n=%zu: %.2fx slower\n", cfg.kernel.c_str(), n, bad / tuned);
        }
    }
    // relativeReport (runner.cpp:303-328): every back-end's median over the baseline's
    if (!cfg.baseline.empty()) {
        std::printf("\nmedian time relative to %s:\n", cfg.baseline.c_str());
        for (std::size_t n : cfg.sizes) {
            const double base = medianOf(cfg.baseline, n, 0);
            if (!(base > 0.0)) {
                std::fprintf(stderr, "kwbench: no '%s' records at n=%zu\n", cfg.baseline.c_str(), n);
                return 2;
            }
            for (const std::string& be : cfg.backends)
                std::printf("  %s %s n=%zu: %.3fx\n", cfg.kernel.c_str(), be.c_str(), n, medianOf(be, n, 0) / base);
        }
    }
    if (!cfg.csv.empty()) {
        std::ofstream os(cfg.csv);
        os << "kernel,backend,n,b,v,tile,rep,seconds,gflops,verified\n";
        for (const auto& r : all)
            os << r.kernel << ',' << r.backend << ',' << r.n << ',' << r.b << ',' << r.v << ',' << r.tile << ','
               << r.rep << ',' << fmt(r.seconds) << ',' << fmt(r.gflops) << ',' << (r.verified ? 1 : 0) << '\n';
    }
    return failed ? 1 : 0;
}
