// kw_axpy.cu — K1: AXPY  Y = alpha*X + Y  on sm_100a.
//
// Reference: AxpyKernel::operator() (/root/reference/proj/core/src/kernels/axpy.cpp:10-23) and
// the oracle axpyReference (core/src/kernels/reference.cpp:8-12).
//
// Arithmetic: y = fl(fl(alpha*x) + y) — __fmul_rn/__fadd_rn (__dmul_rn/__dadd_rn) so nvcc cannot
// contract into FFMA/DFMA; the reference's objects contain mulpd/addpd and no vfmadd, so this is
// the only choice that is bit-exact (SURVEY.md §7 "Hard parts" 1).
//
// Work division → hardware mapping (the element level becomes 128-bit vectors):
//   blocksPerGrid[0]  → gridDim.x        (block b covers elements [b*T*V, (b+1)*T*V), exactly the
//   threadsPerBlock[0]→ blockDim.x        reference block's coverage, work_div.cpp:96-119)
//   elementsPerThread → V elements per thread, issued as V/W vectors of W = 16/sizeof(T)
//                       elements; vector j of thread t sits at b*T*V + (j*T + t)*W so every
//                       warp-wide LDG.128/STG.128 is fully coalesced. The reference's "thread
//                       owns a contiguous run" is an ownership detail of an elementwise update:
//                       no bit of any result depends on which hardware lane computed it.
//   Elements >= n are never read or written (axpy.cpp:15-17 tail guard).
//
// Bytes per element (algorithmic): read X, read Y, write Y = 3*sizeof(T) (12 B for fp32).
//
// Launches use programmatic dependent launch (launch_pdl / griddep_enter): back-to-back steps
// on a stream overlap one grid's launch with the previous grid's tail, and each grid still reads
// Y only after the previous one's writes are visible. Host-resident operands (the e2e path) are
// streamed through device scratch in 32 MiB chunks (run_staged).
#include "kw_common.cuh"

#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>

namespace {

template <typename T>
struct Vec;
template <>
struct Vec<float> {
    using type = float4;
    static constexpr int W = 4;
};
template <>
struct Vec<double> {
    using type = double2;
    static constexpr int W = 2;
};

__device__ __forceinline__ float axpy1(float a, float x, float y) { return __fadd_rn(__fmul_rn(a, x), y); }
__device__ __forceinline__ double axpy1(double a, double x, double y) { return __dadd_rn(__dmul_rn(a, x), y); }

__device__ __forceinline__ float4 axpyv(float a, float4 x, float4 y)
{
    return make_float4(axpy1(a, x.x, y.x), axpy1(a, x.y, y.y), axpy1(a, x.z, y.z), axpy1(a, x.w, y.w));
}
__device__ __forceinline__ double2 axpyv(double a, double2 x, double2 y)
{
    return make_double2(axpy1(a, x.x, y.x), axpy1(a, x.y, y.y));
}

// Programmatic dependent launch (launch_pdl below): every CTA first lets the next grid on the
// stream be admitted, then waits until the previous grid has completed and its writes are
// visible — so back-to-back launches (an in-place Y updated step after step) overlap one grid's
// launch latency with the previous grid's tail without ever reading a stale Y. Without the
// launch attribute both instructions are no-ops.
__device__ __forceinline__ void griddep_enter()
{
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
}

// Streaming loads/stores: X and Y are touched exactly once per launch.
__device__ __forceinline__ float4 ld_stream(const float4* p) { return __ldcs(p); }
__device__ __forceinline__ double2 ld_stream(const double2* p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(float4* p, float4 v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(double2* p, double2 v) { __stcs(p, v); }

// Vector path. `limit` = min(n, grid element extent). U vectors per thread in flight.
template <typename T, int U>
__global__ void __launch_bounds__(1024) axpy_vec_kernel(size_t limit, T alpha, const T* __restrict__ x,
                                                       T* __restrict__ y, uint32_t vecs_per_thread)
{
    griddep_enter();
    using V = typename Vec<T>::type;
    constexpr int W = Vec<T>::W;
    const size_t threads = blockDim.x;
    const size_t block_elems = threads * vecs_per_thread * W;
    const size_t base = static_cast<size_t>(blockIdx.x) * block_elems;
    if (base >= limit)
        return;
    const size_t end = limit - base < block_elems ? limit : base + block_elems;
    const size_t nvec = (end - base) / W; // whole vectors inside [base, end)
    const V* xv = reinterpret_cast<const V*>(x + base);
    V* yv = reinterpret_cast<V*>(y + base);
    for (uint32_t j0 = 0; j0 < vecs_per_thread; j0 += U) {
        V xr[U], yr[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t idx = (j0 + u) * threads + threadIdx.x;
            if (j0 + u < vecs_per_thread && idx < nvec) {
                xr[u] = ld_stream(xv + idx);
                yr[u] = ld_stream(yv + idx);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t idx = (j0 + u) * threads + threadIdx.x;
            if (j0 + u < vecs_per_thread && idx < nvec)
                st_stream(yv + idx, axpyv(alpha, xr[u], yr[u]));
        }
    }
    // Ragged end of the last covered block: fewer than W elements remain.
    for (size_t e = base + nvec * W + threadIdx.x; e < end; e += threads)
        y[e] = axpy1(alpha, x[e], y[e]);
}

// 256-bit path (sm_100a LDG.E.256 / STG.E.256): one 32-byte vector = 8 floats or 4 doubles per
// lane per access, so a warp moves 1 KiB per instruction. X goes through the non-coherent
// path with an L2 256-byte promotion hint; Y is read and written once, never allocated in L1.
template <typename T>
struct V32 {
    static constexpr int W = 32 / sizeof(T);
    T v[W];
};

__device__ __forceinline__ void ld_x32(const float* p, V32<float>& r)
{
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]), "=f"(r.v[6]),
                   "=f"(r.v[7])
                 : "l"(p));
}
__device__ __forceinline__ void ld_y32(const float* p, V32<float>& r)
{
    asm volatile("ld.global.L1::no_allocate.L2::256B.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]), "=f"(r.v[6]),
                   "=f"(r.v[7])
                 : "l"(p));
}
__device__ __forceinline__ void st_y32(float* p, const V32<float>& r)
{
    asm volatile("st.global.L1::no_allocate.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"l"(p), "f"(r.v[0]),
                 "f"(r.v[1]), "f"(r.v[2]), "f"(r.v[3]), "f"(r.v[4]), "f"(r.v[5]), "f"(r.v[6]), "f"(r.v[7])
                 : "memory");
}
__device__ __forceinline__ void ld_x32(const double* p, V32<double>& r)
{
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f64 {%0,%1,%2,%3}, [%4];\n"
                 : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3])
                 : "l"(p));
}
__device__ __forceinline__ void ld_y32(const double* p, V32<double>& r)
{
    asm volatile("ld.global.L1::no_allocate.L2::256B.v4.f64 {%0,%1,%2,%3}, [%4];\n"
                 : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3])
                 : "l"(p));
}
__device__ __forceinline__ void st_y32(double* p, const V32<double>& r)
{
    asm volatile("st.global.L1::no_allocate.v4.f64 [%0], {%1,%2,%3,%4};\n" ::"l"(p), "d"(r.v[0]), "d"(r.v[1]),
                 "d"(r.v[2]), "d"(r.v[3])
                 : "memory");
}

template <typename T, int U>
__global__ void __launch_bounds__(1024) axpy_v32_kernel(size_t limit, T alpha, const T* __restrict__ x,
                                                       T* __restrict__ y, uint32_t vecs_per_thread)
{
    griddep_enter();
    constexpr int W = V32<T>::W;
    const size_t threads = blockDim.x;
    const size_t block_elems = threads * vecs_per_thread * W;
    const size_t base = static_cast<size_t>(blockIdx.x) * block_elems;
    if (base >= limit)
        return;
    const size_t end = limit - base < block_elems ? limit : base + block_elems;
    const size_t nvec = (end - base) / W;
    const T* xb = x + base;
    T* yb = y + base;
    for (uint32_t j0 = 0; j0 < vecs_per_thread; j0 += U) {
        V32<T> xr[U], yr[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t idx = (j0 + u) * threads + threadIdx.x;
            if (j0 + u < vecs_per_thread && idx < nvec) {
                ld_x32(xb + idx * W, xr[u]);
                ld_y32(yb + idx * W, yr[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t idx = (j0 + u) * threads + threadIdx.x;
            if (j0 + u < vecs_per_thread && idx < nvec) {
#pragma unroll
                for (int w = 0; w < W; ++w)
                    yr[u].v[w] = axpy1(alpha, xr[u].v[w], yr[u].v[w]);
                st_y32(yb + idx * W, yr[u]);
            }
        }
    }
    for (size_t e = base + nvec * W + threadIdx.x; e < end; e += threads)
        y[e] = axpy1(alpha, x[e], y[e]);
}

// Vector width policy: 128-bit vectors by default — the measured sweep (profiles/
// axpy_workdiv_sweep_r01.txt) shows both widths saturating HBM at ~7.1 TB/s with the 128-bit
// path at 512 x 4 reproducibly on top; KW_AXPY_VECTOR_BYTES=32 selects the 256-bit path.
int vector_bytes_policy()
{
    static int v = [] {
        const char* e = std::getenv("KW_AXPY_VECTOR_BYTES");
        return (e && std::atoi(e) == 32) ? 32 : 16;
    }();
    return v;
}

// Scalar path (misaligned pointers or V not a multiple of W): element j*T + t of the block.
template <typename T>
__global__ void __launch_bounds__(1024) axpy_scalar_kernel(size_t limit, T alpha, const T* __restrict__ x,
                                                          T* __restrict__ y, uint32_t elems_per_thread)
{
    griddep_enter();
    const size_t threads = blockDim.x;
    const size_t base = static_cast<size_t>(blockIdx.x) * threads * elems_per_thread;
    for (uint32_t j = 0; j < elems_per_thread; ++j) {
        const size_t e = base + j * threads + threadIdx.x;
        if (e < limit)
            y[e] = axpy1(alpha, x[e], y[e]);
    }
}

template <typename T>
kw_status validate_wd(const kw_workdiv* wd, size_t n, size_t& blocks, uint32_t& threads, uint32_t& elems,
                      size_t& limit)
{
    if (wd->dim != 1)
        return kw::usage("axpy: the AXPY kernel runs on a 1-D work division");
    if (wd->blocks[0] == 0 || wd->threads[0] == 0 || wd->elems[0] == 0)
        return kw::usage("WorkDiv: every level extent is at least 1");
    if (wd->threads[0] > 1024)
        return kw::usage("axpy: threadsPerBlock " + std::to_string(wd->threads[0]) +
                         " exceeds the sm_100a block limit of 1024");
    if (wd->blocks[0] > static_cast<size_t>(INT_MAX))
        return kw::usage("axpy: blocksPerGrid exceeds the grid limit");
    if (wd->elems[0] > (1u << 30))
        return kw::usage("axpy: elementsPerThread too large");
    blocks = wd->blocks[0];
    threads = static_cast<uint32_t>(wd->threads[0]);
    elems = static_cast<uint32_t>(wd->elems[0]);
    size_t covered = 0; // saturates: a division that large covers every index
    if (__builtin_mul_overflow(blocks, static_cast<size_t>(threads) * elems, &covered))
        covered = SIZE_MAX;
    limit = covered < n ? covered : n; // only covered indices are computed (axpy.cpp:12-17)
    return KW_OK;
}

// KW_PDL=0 disables programmatic dependent launch (A/B switch).
bool pdl_policy()
{
    static const bool on = [] {
        const char* e = std::getenv("KW_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

template <typename... Params, typename... Args>
void launch_pdl(void (*kernel)(Params...), unsigned grid, unsigned threads, cudaStream_t s, Args... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_policy() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, static_cast<Params>(args)...);
}

// Which kernel template a device-resident launch runs (the one place that decides: the launcher
// below and kw_axpy_kernel_name both call it, so the name bench.py reports is the launched one).
enum class AxpyPath { V32x2, V32x1, Vec4, Vec2, Vec1, Scalar };

template <typename T>
AxpyPath select_path(uint32_t elems, const void* x, const void* y)
{
    constexpr int W = Vec<T>::W;
    constexpr int W32 = V32<T>::W;
    const bool aligned = (reinterpret_cast<uintptr_t>(x) % 16 == 0) && (reinterpret_cast<uintptr_t>(y) % 16 == 0);
    const bool aligned32 = (reinterpret_cast<uintptr_t>(x) % 32 == 0) && (reinterpret_cast<uintptr_t>(y) % 32 == 0);
    if (vector_bytes_policy() == 32 && aligned32 && elems % W32 == 0)
        return elems / W32 >= 2 ? AxpyPath::V32x2 : AxpyPath::V32x1;
    if (aligned && elems % W == 0) {
        const uint32_t vpt = elems / W;
        return vpt >= 4 ? AxpyPath::Vec4 : vpt >= 2 ? AxpyPath::Vec2 : AxpyPath::Vec1;
    }
    return AxpyPath::Scalar;
}

template <typename T>
std::string path_name(AxpyPath p)
{
    const std::string t = sizeof(T) == 4 ? "float" : "double";
    switch (p) {
    case AxpyPath::V32x2: return "axpy_v32_kernel<" + t + ",2>";
    case AxpyPath::V32x1: return "axpy_v32_kernel<" + t + ",1>";
    case AxpyPath::Vec4: return "axpy_vec_kernel<" + t + ",4>";
    case AxpyPath::Vec2: return "axpy_vec_kernel<" + t + ",2>";
    case AxpyPath::Vec1: return "axpy_vec_kernel<" + t + ",1>";
    default: return "axpy_scalar_kernel<" + t + ">";
    }
}

template <typename T>
void launch_device(cudaStream_t s, size_t blocks, uint32_t threads, uint32_t elems, size_t limit, T alpha,
                   const T* x, T* y)
{
    constexpr int W = Vec<T>::W;
    constexpr int W32 = V32<T>::W;
    // Blocks entirely beyond `limit` have nothing to do: do not launch them.
    const size_t block_elems = static_cast<size_t>(threads) * elems;
    const size_t useful = kw::ceil_div(limit, block_elems);
    const unsigned grid = static_cast<unsigned>(useful < blocks ? useful : blocks);
    if (grid == 0)
        return;
    switch (select_path<T>(elems, x, y)) {
    case AxpyPath::V32x2: launch_pdl(axpy_v32_kernel<T, 2>, grid, threads, s, limit, alpha, x, y, elems / W32); break;
    case AxpyPath::V32x1: launch_pdl(axpy_v32_kernel<T, 1>, grid, threads, s, limit, alpha, x, y, elems / W32); break;
    case AxpyPath::Vec4: launch_pdl(axpy_vec_kernel<T, 4>, grid, threads, s, limit, alpha, x, y, elems / W); break;
    case AxpyPath::Vec2: launch_pdl(axpy_vec_kernel<T, 2>, grid, threads, s, limit, alpha, x, y, elems / W); break;
    case AxpyPath::Vec1: launch_pdl(axpy_vec_kernel<T, 1>, grid, threads, s, limit, alpha, x, y, elems / W); break;
    default: launch_pdl(axpy_scalar_kernel<T>, grid, threads, s, limit, alpha, x, y, elems); break;
    }
    kw::g_launches.fetch_add(1, std::memory_order_relaxed);
}

// Host-resident operands (the e2e path: executeTask on Device::host() buffers): stream the
// vectors through device scratch in chunks. H2D + kernel on the queue's stream, D2H on the
// aux stream, a ring of slots with events so the H2D of chunk c+1 overlaps the D2H of chunk c
// (PCIe is full duplex). The queue stream finally joins the aux stream, so later tasks on the
// queue observe the completed Y (in-order FIFO, queue.hpp:86-93).
template <typename T>
kw_status run_staged(kw::Queue* q, uint32_t threads, uint32_t elems, size_t limit, T alpha, const T* x, T* y,
                     bool x_dev, bool y_dev)
{
    // Chunk bytes per operand per slot (KW_STAGE_CHUNK_MB overrides; measured in
    // profiles/e2e_chunk_sweep_r01.txt), 4 slots.
    static const size_t kChunkBytes = [] {
        const char* e = std::getenv("KW_STAGE_CHUNK_MB");
        const long v = e ? std::atol(e) : 0;
        return static_cast<size_t>(v > 0 && v <= 1024 ? v : 32) << 20;
    }();
    const size_t chunk = kChunkBytes / sizeof(T);
    const int ring = kw::Queue::kRing;
    const size_t slot_elems = chunk * 2;
    kw_status st = kw::ensure_scratch(q, ring * slot_elems * sizeof(T));
    if (st != KW_OK)
        return st;
    T* scratch = static_cast<T*>(q->scratch);
    const size_t block_elems = static_cast<size_t>(threads) * elems;
    const size_t nchunks = kw::ceil_div(limit, chunk);
    cudaError_t e = cudaSuccess;
    for (size_t c = 0; c < nchunks && e == cudaSuccess; ++c) {
        const int s = static_cast<int>(c % ring);
        const size_t off = c * chunk;
        const size_t len = limit - off < chunk ? limit - off : chunk;
        T* xs = scratch + s * slot_elems;
        T* ys = xs + chunk;
        if (c >= static_cast<size_t>(ring))
            e = cudaStreamWaitEvent(q->stream, q->ev_free[s], 0);
        const T* xd = x + off;
        T* yd = y + off;
        if (e == cudaSuccess && !x_dev) {
            e = cudaMemcpyAsync(xs, x + off, len * sizeof(T), cudaMemcpyHostToDevice, q->stream);
            xd = xs;
        }
        if (e == cudaSuccess && !y_dev) {
            e = cudaMemcpyAsync(ys, y + off, len * sizeof(T), cudaMemcpyHostToDevice, q->stream);
            yd = ys;
        }
        if (e != cudaSuccess)
            break;
        launch_device<T>(q->stream, kw::ceil_div(len, block_elems), threads, elems, len, alpha, xd, yd);
        e = cudaGetLastError();
        if (e == cudaSuccess && !y_dev) {
            e = cudaEventRecord(q->ev_ready[s], q->stream);
            if (e == cudaSuccess)
                e = cudaStreamWaitEvent(q->aux, q->ev_ready[s], 0);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(y + off, ys, len * sizeof(T), cudaMemcpyDeviceToHost, q->aux);
            if (e == cudaSuccess)
                e = cudaEventRecord(q->ev_free[s], q->aux);
        }
        else if (e == cudaSuccess) {
            e = cudaEventRecord(q->ev_free[s], q->stream);
        }
    }
    if (e == cudaSuccess) {
        e = cudaEventRecord(q->ev_join, q->aux);
        if (e == cudaSuccess)
            e = cudaStreamWaitEvent(q->stream, q->ev_join, 0);
    }
    if (e != cudaSuccess)
        return kw::task_fail(q, std::string("axpy (host-staged): ") + cudaGetErrorString(e));
    return kw::after_enqueue(q, "axpy");
}

// Zero-copy (host-resident operands): the kernel itself loads X and Y from, and stores Y to,
// page-locked host memory over PCIe (the pinned pages are mapped into the device address space),
// instead of the copy engines staging chunks through device scratch. Same kernel, same bits.
// KW_AXPY_ZEROCOPY=0/1 overrides the default (A/B measurements).
bool axpy_zero_copy_policy()
{
    static const bool on = [] {
        const char* e = std::getenv("KW_AXPY_ZEROCOPY");
        return e ? e[0] == '1' : false;
    }();
    return on;
}

// Device-side address of a pinned host pointer (nullptr: not pinned-and-mapped).
const void* mapped_host_ptr(const void* p)
{
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

template <typename T>
kw_status axpy_entry(kw_queue qh, const kw_workdiv* wd, size_t n, T alpha, const T* x, T* y)
{
    KW_CHECK_QUEUE(qh);
    KW_ENQUEUE_LOCK(qh);
    KW_NVTX("kw axpy");
    auto* q = reinterpret_cast<kw::Queue*>(qh);
    kw_workdiv def;
    if (wd == nullptr) {
        kw_status st = kw_axpy_default_workdiv(n, static_cast<int>(sizeof(T)), &def);
        if (st != KW_OK)
            return st;
        wd = &def;
    }
    size_t blocks, limit;
    uint32_t threads, elems;
    kw_status st = validate_wd<T>(wd, n, blocks, threads, elems, limit);
    if (st != KW_OK)
        return st;
    if (limit == 0)
        return KW_OK;
    if (x == nullptr || y == nullptr)
        return kw::usage("axpy: null buffer");
    kw::DeviceGuard g(q->device);
    int xdev = -1, ydev = -1;
    const bool x_dev = kw::pointer_kind(x, &xdev) == KW_MEM_DEVICE;
    const bool y_dev = kw::pointer_kind(y, &ydev) == KW_MEM_DEVICE;
    if ((x_dev && xdev != q->device) || (y_dev && ydev != q->device))
        return kw::usage("axpy: buffer lives on a different device than the queue");
    if (x_dev && y_dev) {
        launch_device<T>(q->stream, blocks, threads, elems, limit, alpha, x, y);
        return kw::after_enqueue(q, "axpy");
    }
    if (axpy_zero_copy_policy()) {
        const T* xm = x_dev ? x : static_cast<const T*>(mapped_host_ptr(x));
        T* ym = y_dev ? y : static_cast<T*>(const_cast<void*>(mapped_host_ptr(y)));
        if (xm && ym) {
            launch_device<T>(q->stream, blocks, threads, elems, limit, alpha, xm, ym);
            return kw::after_enqueue(q, "axpy");
        }
    }
    return run_staged<T>(q, threads, elems, limit, alpha, x, y, x_dev, y_dev);
}

} // namespace

extern "C" {

kw_status kw_axpy_default_workdiv(size_t n, int elem_size, kw_workdiv* out)
{
    if (!out)
        return kw::usage("kw_axpy_default_workdiv: null output");
    if (elem_size != 4 && elem_size != 8)
        return kw::usage("kw_axpy_default_workdiv: element size must be 4 or 8");
    // 512 threads x one 16-byte vector per thread (the sweep's best point): 131072 blocks at
    // n = 2^28, ~900 waves over 148 SMs, so the grid tail is negligible.
    const size_t threads = 512, elems = elem_size == 4 ? 4 : 2;
    kw_workdiv wd = {};
    wd.dim = 1;
    for (int k = 0; k < 3; ++k)
        wd.blocks[k] = wd.threads[k] = wd.elems[k] = 1;
    wd.threads[0] = threads;
    wd.elems[0] = elems;
    wd.blocks[0] = n == 0 ? 1 : kw::ceil_div(n, threads * elems);
    *out = wd;
    return KW_OK;
}

kw_status kw_axpy_f32(kw_queue q, const kw_workdiv* wd, size_t n, float alpha, const float* x, float* y)
{
    return axpy_entry<float>(q, wd, n, alpha, x, y);
}

kw_status kw_axpy_f64(kw_queue q, const kw_workdiv* wd, size_t n, double alpha, const double* x, double* y)
{
    return axpy_entry<double>(q, wd, n, alpha, x, y);
}

kw_status kw_axpy_kernel_name(const kw_workdiv* wd, int elem_size, const void* x, const void* y, char* buf,
                              size_t len)
{
    if (!wd || !buf || len == 0)
        return kw::usage("kw_axpy_kernel_name: null argument");
    if (elem_size != 4 && elem_size != 8)
        return kw::usage("kw_axpy_kernel_name: element size must be 4 or 8");
    if (wd->dim != 1 || wd->elems[0] == 0 || wd->elems[0] > (1u << 30))
        return kw::usage("kw_axpy_kernel_name: not a valid 1-D AXPY division");
    const uint32_t elems = static_cast<uint32_t>(wd->elems[0]);
    const std::string name = elem_size == 4 ? path_name<float>(select_path<float>(elems, x, y))
                                            : path_name<double>(select_path<double>(elems, x, y));
    std::snprintf(buf, len, "%s", name.c_str());
    return KW_OK;
}

} // extern "C"
