// Per-task overhead of the library path vs a native launch, tiny AXPY (kernel ~2 us).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++20 -I include overhead.cu -L.. -lkw_b200
#include <kernelweave/kernelweave.hpp>

#include <chrono>
#include <cstdio>

using namespace kernelweave;
using namespace kernelweave::kernels;
using Clock = std::chrono::steady_clock;

__global__ void native_axpy(std::size_t n, double a, const double* x, double* y)
{
    const std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n)
        y[i] = __dadd_rn(__dmul_rn(a, x[i]), y[i]);
}

template <class F>
double per_call_us(F&& f, int reps = 2000)
{
    for (int i = 0; i < 50; ++i)
        f();
    const auto t0 = Clock::now();
    for (int i = 0; i < reps; ++i)
        f();
    return std::chrono::duration<double, std::micro>(Clock::now() - t0).count() / reps;
}

int main()
{
    const std::size_t n = 1 << 20;
    Buffer x(Device::gpu(0), IndexVec(n), 8), y(Device::gpu(0), IndexVec(n), 8);
    Queue sq(Device::gpu(0), QueueFlavor::Sync), aq(Device::gpu(0), QueueFlavor::Async);
    kw_memset(sq.native(), x.data(), 0, n * 8);
    kw_memset(sq.native(), y.data(), 0, n * 8);
    void* sp = nullptr;
    kw_queue_stream(aq.native(), &sp);
    cudaStream_t s = static_cast<cudaStream_t>(sp);
    double* xd = x.rowData<double>(0);
    double* yd = y.rowData<double>(0);
    const WorkDiv wd = axpyWorkDiv(BackendKind::GpuCudaRt, n, 512, 4);
    const kw_workdiv w = wd.toC();
    std::printf("native launch + cudaStreamSynchronize : %6.2f us\n", per_call_us([&] {
        native_axpy<<<(n + 255) / 256, 256, 0, s>>>(n, 0.5, xd, yd);
        cudaStreamSynchronize(s);
    }));
    std::printf("native launch only (async)            : %6.2f us\n", per_call_us([&] {
        native_axpy<<<(n + 255) / 256, 256, 0, s>>>(n, 0.5, xd, yd);
    }));
    cudaStreamSynchronize(s);
    std::printf("C-ABI kw_axpy_f64 (async) + wait      : %6.2f us\n", per_call_us([&] {
        kw_axpy_f64(aq.native(), &w, n, 0.5, xd, yd);
        kw_queue_wait(aq.native());
    }));
    std::printf("C-ABI kw_axpy_f64 (async) only        : %6.2f us\n", per_call_us([&] {
        kw_axpy_f64(aq.native(), &w, n, 0.5, xd, yd);
    }));
    kw_queue_wait(aq.native());
    std::printf("kw_queue_wait on idle queue           : %6.2f us\n", per_call_us([&] { kw_queue_wait(aq.native()); }));
    std::printf("kw_event_record + destroy             : %6.2f us\n", per_call_us([&] {
        kw_event ev = nullptr;
        kw_event_record(aq.native(), &ev);
        kw_event_destroy(ev);
    }));
    std::printf("kw_task_marker + destroy              : %6.2f us\n", per_call_us([&] {
        kw_event ev = nullptr;
        kw_task_marker(aq.native(), &ev);
        kw_event_destroy(ev);
    }));
    std::printf("C-ABI kw_axpy_f64 (Sync queue)        : %6.2f us\n", per_call_us([&] {
        kw_axpy_f64(sq.native(), &w, n, 0.5, xd, yd);
    }));
    std::printf("  + kw_event_record/destroy           : %6.2f us\n", per_call_us([&] {
        kw_axpy_f64(sq.native(), &w, n, 0.5, xd, yd);
        kw_event ev = nullptr;
        kw_event_record(sq.native(), &ev);
        kw_event_destroy(ev);
    }));
    std::printf("  + kw_queue_wait                     : %6.2f us\n", per_call_us([&] {
        kw_axpy_f64(sq.native(), &w, n, 0.5, xd, yd);
        kw_event ev = nullptr;
        kw_event_record(sq.native(), &ev);
        kw_event_destroy(ev);
        kw_queue_wait(sq.native());
    }));
    std::printf("createExec only (no enqueue)          : %6.2f us\n", per_call_us([&] {
        ExecTask t = createExec(BackendKind::GpuCudaRt, wd, AxpyKernel{}, AxpyArgs{n, 0.5, &x, &y});
        (void)t;
    }));
    std::printf("C++ Queue(Async).enqueue + wait       : %6.2f us\n", per_call_us([&] {
        aq.enqueue(createExec(BackendKind::GpuCudaRt, wd, AxpyKernel{}, AxpyArgs{n, 0.5, &x, &y}));
        aq.wait();
    }));
    std::printf("C++ Queue(Sync).enqueue + wait        : %6.2f us\n", per_call_us([&] {
        sq.enqueue(createExec(BackendKind::GpuCudaRt, wd, AxpyKernel{}, AxpyArgs{n, 0.5, &x, &y}));
        sq.wait();
    }));
    std::printf("C++ executeTask                       : %6.2f us\n", per_call_us([&] {
        executeTask(BackendKind::GpuCudaRt, wd, AxpyKernel{}, AxpyArgs{n, 0.5, &x, &y});
    }));
    return 0;
}
