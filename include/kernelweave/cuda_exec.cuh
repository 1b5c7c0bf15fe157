/* kernelweave B200 drop-in — generic device functor launch.
 *
 * Runs ANY kernelweave functor `operator()(const AccContext&, Args...)` on the GPU, the role
 * detail::runGrid plays for the reference's CPU engines (accel.cpp:120-265): one CUDA thread per
 * (block, thread) pair of the work division, the last (fastest) work-division component on
 * CUDA x. Inside the functor the reference's kernel-side API works unchanged:
 *   getIdx / getWorkDiv (both spellings)        -> acc.hpp (host/device)
 *   allocSharedMem<T>(acc, n)                   -> dynamic shared memory, matched by call
 *                                                  sequence, zero-initialised (accel.cpp:286-292)
 *   syncBlockThreads(acc)                       -> __syncthreads (accel.cpp:294-302)
 *   atomicAdd(acc, cell, v) f64 / i64 / u64     -> native global atomics (accel.cpp:304-321)
 *   failTask(acc, code)                         -> the device form of throwing from a functor
 *                                                  (accel.cpp:240-248): the task fails, wait()
 *                                                  raises TaskError, later tasks still run
 * Buffers cross into device code as BufferView (pointer, pitch, extent): a host Buffer object
 * cannot be dereferenced on the GPU.
 *
 * Usage (translation unit compiled by nvcc -gencode arch=compute_100a,code=sm_100a):
 *   struct MyKernel { template <class Acc> __device__ void operator()(const Acc&, Args) const; };
 *   KW_DEVICE_FUNCTOR(MyKernel)          // at global scope
 *   executeTask(BackendKind::GpuCudaRt, wd, MyKernel{}, args...);
 * A functor may declare `static constexpr std::size_t sharedMemBytes = …;` (default 48 KiB).
 */
#pragma once

#if !defined(__CUDACC__)
#error "kernelweave/cuda_exec.cuh must be compiled by nvcc"
#endif

#include "kernelweave/kernelweave.hpp"

#include <cuda_runtime.h>

#include <cstdint>

namespace kernelweave {

/// Device view of a Buffer (buffer.hpp:29-128 accessors that make sense on the GPU).
struct BufferView {
    std::byte* ptr = nullptr;
    std::size_t pitch = 0;
    std::size_t elemSize = 0;
    std::uint32_t dim = 1;
    std::size_t extent[3] = {1, 1, 1};
    int device = 0;

    template <class T>
    __host__ __device__ T* rowData(std::size_t row) const noexcept
    {
        return reinterpret_cast<T*>(ptr + row * pitch);
    }
    template <class T>
    __host__ __device__ std::size_t leadingDim() const noexcept
    {
        return pitch / sizeof(T);
    }
    __host__ __device__ std::size_t rowCount() const noexcept
    {
        std::size_t r = 1;
        for (std::uint32_t k = 0; k + 1 < dim; ++k)
            r *= extent[k];
        return r;
    }
};

inline BufferView view(const Buffer& b)
{
    if (b.device().isHost())
        throw UsageError("BufferView: device functors take GPU buffers (copy host data first)");
    BufferView v;
    v.ptr = const_cast<std::byte*>(b.data());
    v.pitch = b.rowPitch();
    v.elemSize = b.elemSize();
    v.dim = static_cast<std::uint32_t>(b.dim());
    for (std::size_t k = 0; k < b.dim(); ++k)
        v.extent[k] = b.extent()[k];
    v.device = b.device().cudaIndex();
    return v;
}

/// Fails the running task with a non-zero code (any thread, any number of times; one code is
/// kept). Device code cannot throw, so the functor returns after calling this — the reference's
/// `throw` inside operator() (test_accel.cpp:403-430). Reported by Queue::wait() as TaskError and
/// by the task's TaskHandle as TaskState::Failed; later tasks on the queue still run.
__device__ inline void failTask(const AccContext& acc, unsigned code = 1)
{
    if (std::uint32_t* s = acc.failSlot())
        *reinterpret_cast<volatile std::uint32_t*>(s) = code ? code : 1u;
}

/// Block-shared region of count*elemSize bytes; every thread of the block must issue the same
/// allocation sequence (acc.hpp:75-84 contract), which makes this a collective: the region is
/// zeroed cooperatively and published with a block barrier.
__device__ inline void* allocSharedMem(const AccContext& acc, std::size_t elemCount, std::size_t elemSize)
{
    const std::size_t bytes = elemCount * elemSize;
    const std::size_t off = (acc.sharedCursor() + 15) & ~static_cast<std::size_t>(15);
    if (bytes == 0 || off + bytes > acc.sharedBytes()) {
        // The reference throws UsageError out of operator() (accel.cpp:286-292): the task fails,
        // the queue and later tasks live on. Here the allocation sequence is block-uniform, so
        // every thread of the block takes this branch: record the failure and retire the block
        // (the functor body never runs past the failed allocation). No trap — a trap would
        // poison the CUDA context for every queue in the process.
        failTask(acc, KW_FAIL_SHARED_OVERFLOW);
        asm volatile("exit;");
    }
    acc.sharedCursor() = off + bytes;
    std::byte* p = acc.sharedBase() + off;
    const unsigned nthreads = blockDim.x * blockDim.y * blockDim.z;
    const unsigned tid = (threadIdx.z * blockDim.y + threadIdx.y) * blockDim.x + threadIdx.x;
    for (std::size_t i = tid; i < bytes; i += nthreads)
        p[i] = std::byte{0};
    __syncthreads();
    return p;
}

template <class T>
__device__ inline T* allocSharedMem(const AccContext& acc, std::size_t count)
{
    return static_cast<T*>(allocSharedMem(acc, count, sizeof(T)));
}

__device__ inline void syncBlockThreads(const AccContext&) { __syncthreads(); }

__device__ inline double atomicAdd(const AccContext&, double& cell, double operand)
{
    return ::atomicAdd(&cell, operand);
}
__device__ inline std::int64_t atomicAdd(const AccContext&, std::int64_t& cell, std::int64_t operand)
{
    return static_cast<std::int64_t>(::atomicAdd(reinterpret_cast<unsigned long long*>(&cell),
                                                 static_cast<unsigned long long>(operand)));
}
__device__ inline std::uint64_t atomicAdd(const AccContext&, std::uint64_t& cell, std::uint64_t operand)
{
    return static_cast<std::uint64_t>(::atomicAdd(reinterpret_cast<unsigned long long*>(&cell),
                                                 static_cast<unsigned long long>(operand)));
}

namespace detail {

template <class Kernel, class = void>
struct SharedBytesOf {
    static constexpr std::size_t value = 48 * 1024;
};
template <class Kernel>
struct SharedBytesOf<Kernel, std::void_t<decltype(Kernel::sharedMemBytes)>> {
    static constexpr std::size_t value = Kernel::sharedMemBytes;
};

/// Logical blocks of a division, and logical block `lb` (row-major, last component fastest —
/// delinearize of index_vec.hpp) as the device computes it for every functor launch. Scalar,
/// array-free. Pinned exhaustively on the device by acceptance criterion 03's extent set
/// (tests/cpp/test_functor_gpu.cu).
KW_HD inline std::size_t logicalBlockCount(const kw_workdiv& wd) noexcept
{
    const unsigned d = wd.dim;
    return wd.blocks[d - 1] * (d >= 2 ? wd.blocks[d - 2] : 1) * (d == 3 ? wd.blocks[0] : 1);
}
KW_HD inline IndexVec logicalBlockIdx(const kw_workdiv& wd, std::size_t lb) noexcept
{
    const unsigned d = wd.dim;
    const std::size_t bLast = wd.blocks[d - 1], bMid = d >= 2 ? wd.blocks[d - 2] : 1;
    const std::size_t c = lb % bLast, r = lb / bLast;
    return d == 1 ? IndexVec(c) : d == 2 ? IndexVec(r, c) : IndexVec(r / bMid, r % bMid, c);
}

template <class Kernel, class... Args>
__global__ void functorKernel(kw_workdiv wd, std::size_t sharedBytes, std::uint32_t* failSlot, Kernel kernel,
                              Args... args)
{
    extern __shared__ __align__(16) std::byte kwSharedArena[];
    // Logical blocks lb = blockIdx.x, +gridDim.x, ... (one per CUDA block unless the division has
    // more than 2^31-1 blocks, when a resident grid walks them). Last work-division component =
    // fastest (index_vec.hpp:15-24). Built
    // from scalars: local index arrays here were once assigned one stack slot by nvcc 12.9 (the
    // block index read back as the thread index) — keep this path array-free.
    const unsigned d = wd.dim;
    const IndexVec tIdx = d == 1 ? IndexVec(threadIdx.x)
                          : d == 2 ? IndexVec(threadIdx.y, threadIdx.x)
                                   : IndexVec(threadIdx.z, threadIdx.y, threadIdx.x);
    const std::size_t nb = logicalBlockCount(wd);
    for (std::size_t lb = blockIdx.x; lb < nb; lb += gridDim.x) {
        const AccContext acc(wd, logicalBlockIdx(wd, lb), tIdx, kwSharedArena, sharedBytes, failSlot);
        kernel(acc, args...);
        if (lb + gridDim.x < nb)
            __syncthreads(); // the next logical block reuses the shared arena
    }
}

template <class T>
int viewDevice(const T&)
{
    return -1;
}
inline int viewDevice(const BufferView& v) { return v.device; }

template <class Kernel, class... Args>
struct DeviceLauncher {
    static dim3 toDim3(const std::size_t* v, std::uint32_t d)
    {
        return dim3(static_cast<unsigned>(v[d - 1]), d >= 2 ? static_cast<unsigned>(v[d - 2]) : 1u,
                    d == 3 ? static_cast<unsigned>(v[0]) : 1u);
    }
    static void validate(const WorkDiv& wd, const Args&...)
    {
        const kw_workdiv w = wd.toC();
        std::size_t threads = 1;
        for (std::uint32_t k = 0; k < w.dim; ++k)
            threads *= w.threads[k];
        if (threads > 1024)
            throw UsageError("device functor: threadsPerBlock exceeds the sm_100a block limit of 1024");
        if (w.elems[0] * w.elems[1] * w.elems[2] == 0)
            throw UsageError("WorkDiv: every level extent is at least 1");
    }
    static kw_status launch(kw_queue q, const WorkDiv& wd, const Kernel& kernel, const Args&... args)
    {
        void* stream = nullptr;
        int dev = 0;
        std::uint32_t* failSlot = nullptr;
        // One enqueue: begin takes the queue's enqueue lock (FIFO against concurrent enqueues,
        // rejects a shut-down queue); end arms the failure slot and releases the lock.
        kw_status st = kw_queue_begin_launch(q, "device functor", &stream, &dev, &failSlot);
        if (st != KW_OK)
            return st;
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(dev);
        const kw_workdiv w = wd.toC();
        constexpr std::size_t smem = SharedBytesOf<Kernel>::value;
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(functorKernel<Kernel, Args...>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem));
        // Logical blocks -> CUDA blocks on a 1-D grid (2-D/3-D divisions are linearised, so
        // CUDA's 65535 limit on y/z never applies). A division up to 32 resident waves deep gets
        // one CUDA block per logical block — the hardware scheduler balances them (the paper's
        // tiled DGEMM: 100 % of the native kernel). Deeper divisions (or more than 2^31-1 blocks)
        // run on one resident wave of CUDA blocks, each walking >= 32 logical blocks, so block
        // launches stop dominating short blocks at <= 3 % static imbalance (the README AXPY
        // functor at 1024 x 2: 0.29 ms walking vs 0.51 ms one-per-block).
        std::size_t nb = 1;
        for (std::uint32_t k = 0; k < w.dim; ++k)
            nb *= w.blocks[k];
        const dim3 block = toDim3(w.threads, w.dim);
        const int threads = static_cast<int>(block.x * block.y * block.z);
        static thread_local int cachedThreads = -1, cachedDev = -1;
        static thread_local std::size_t cachedResident = 0;
        if (cachedThreads != threads || cachedDev != dev) {
            int perSm = 0, sms = 0;
            if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) {
                cudaGetLastError();
                sms = 148;
            }
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&perSm, functorKernel<Kernel, Args...>, threads, smem) !=
                cudaSuccess) {
                cudaGetLastError(); // e.g. a block that cannot fit: the launch itself reports it
                perSm = 1;
            }
            cachedResident = static_cast<std::size_t>(perSm > 0 ? perSm : 1) * static_cast<std::size_t>(sms);
            cachedThreads = threads;
            cachedDev = dev;
        }
        const std::size_t resident = cachedResident;
        const std::size_t grid_blocks = (nb > 32 * resident || nb > 2147483647u) ? resident : nb;
        const unsigned grid = static_cast<unsigned>(grid_blocks);
        functorKernel<Kernel, Args...><<<grid, block, smem, static_cast<cudaStream_t>(stream)>>>(w, smem, failSlot,
                                                                                                kernel, args...);
        const int err = static_cast<int>(cudaGetLastError());
        st = kw_queue_end_launch(q, err, "device functor");
        cudaSetDevice(prev);
        return st;
    }
    static Device device(const Args&... args)
    {
        int d = -1;
        ((d = d >= 0 ? d : viewDevice(args)), ...);
        return Device::gpu(d >= 0 ? d : 0);
    }
};

} // namespace detail
} // namespace kernelweave

/// Registers a user functor for GPU execution through createExec / executeTask.
#define KW_DEVICE_FUNCTOR(K)                                                                                   \
    namespace kernelweave::detail {                                                                            \
    template <class... Args>                                                                                   \
    struct Launcher<K, Args...> : DeviceLauncher<K, Args...> {                                                 \
    };                                                                                                         \
    }
