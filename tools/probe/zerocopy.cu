// Zero-copy probe: can SM loads/stores to mapped pinned host memory move AXPY's 2:1 H2D:D2H byte
// mix faster than the copy engines (78.8 GB/s, pcie.cu)? Y = a*X + Y with X, Y in pinned host
// memory: (1) copy engines only (reference point), (2) kernel reads X, Y and writes Y over PCIe,
// (3) read-only and write-only kernels (one direction each), (4) copy-engine H2D + kernel-store D2H.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o zerocopy zerocopy.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int U>
__global__ void __launch_bounds__(512) axpy_zc(size_t n4, float a, const float4* __restrict__ x, float4* y)
{
    const size_t stride = size_t(gridDim.x) * blockDim.x * U;
    for (size_t i = size_t(blockIdx.x) * blockDim.x * U + threadIdx.x; i < n4; i += stride) {
        float4 xv[U], yv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t j = i + size_t(u) * blockDim.x;
            if (j < n4) {
                xv[u] = x[j];
                yv[u] = y[j];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t j = i + size_t(u) * blockDim.x;
            if (j < n4) {
                float4 r;
                r.x = __fadd_rn(__fmul_rn(a, xv[u].x), yv[u].x);
                r.y = __fadd_rn(__fmul_rn(a, xv[u].y), yv[u].y);
                r.z = __fadd_rn(__fmul_rn(a, xv[u].z), yv[u].z);
                r.w = __fadd_rn(__fmul_rn(a, xv[u].w), yv[u].w);
                y[j] = r;
            }
        }
    }
}

template <int U>
__global__ void __launch_bounds__(512) read_zc(size_t n4, const float4* __restrict__ x, float* out)
{
    const size_t stride = size_t(gridDim.x) * blockDim.x * U;
    float acc = 0.f;
    for (size_t i = size_t(blockIdx.x) * blockDim.x * U + threadIdx.x; i < n4; i += stride) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t j = i + size_t(u) * blockDim.x;
            v[u] = j < n4 ? x[j] : make_float4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            acc += v[u].x + v[u].y + v[u].z + v[u].w;
    }
    if (acc == 1234.5f)
        out[0] = acc;
}

__global__ void __launch_bounds__(512) write_zc(size_t n4, float4* y, const float4* __restrict__ src)
{
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride)
        y[i] = src[i];
}

int main()
{
    const size_t n = size_t(1) << 28, bytes = n * 4, n4 = n / 4;
    float *hx, *hy, *dx, *dy, *dout;
    cudaHostAlloc(&hx, bytes, cudaHostAllocMapped);
    cudaHostAlloc(&hy, bytes, cudaHostAllocMapped);
    cudaMalloc(&dx, bytes);
    cudaMalloc(&dy, bytes);
    cudaMalloc(&dout, 64);
    for (size_t i = 0; i < n; ++i) {
        hx[i] = 1.0f;
        hy[i] = 2.0f;
    }
    float *mx, *my;
    cudaHostGetDevicePointer(&mx, hx, 0);
    cudaHostGetDevicePointer(&my, hy, 0);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaStream_t s[3];
    for (auto& x : s)
        cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, auto&& body, double total) {
        body();
        cudaDeviceSynchronize();
        float best = 1e30f, sum = 0;
        const int reps = 5;
        for (int r = 0; r < reps; ++r) {
            cudaDeviceSynchronize();
            cudaEventRecord(e0, 0);
            body();
            cudaDeviceSynchronize();
            cudaEventRecord(e1, 0);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
            sum += ms;
        }
        cudaError_t err = cudaGetLastError();
        std::printf("%-52s best %7.2f ms %6.1f GB/s  mean %6.1f GB/s %s\n", name, best, total / best / 1e6,
                    total / (sum / reps) / 1e6, err == cudaSuccess ? "" : cudaGetErrorString(err));
    };
    const double mix = 3.0 * bytes;
    run("copy engines: H2D X, Y + D2H Y (2 streams)", [&] {
        cudaMemcpyAsync(dx, hx, bytes, cudaMemcpyHostToDevice, s[0]);
        cudaMemcpyAsync(dy, hy, bytes, cudaMemcpyHostToDevice, s[1]);
        cudaMemcpyAsync(hy, dy, bytes, cudaMemcpyDeviceToHost, s[2]);
    }, mix);
    for (int bps : {1, 2, 4, 8}) {
        char name[96];
        std::snprintf(name, sizeof name, "zero-copy AXPY U=4, %d blocks/SM x 512", bps);
        run(name, [&] { axpy_zc<4><<<sms * bps, 512, 0, s[0]>>>(n4, 1.5f, (const float4*)mx, (float4*)my); }, mix);
    }
    run("zero-copy AXPY U=8, 4 blocks/SM x 512",
        [&] { axpy_zc<8><<<sms * 4, 512, 0, s[0]>>>(n4, 1.5f, (const float4*)mx, (float4*)my); }, mix);
    run("zero-copy read X (H2D by SM loads), U=8, 4 blocks/SM",
        [&] { read_zc<8><<<sms * 4, 512, 0, s[0]>>>(n4, (const float4*)mx, dout); }, double(bytes));
    run("zero-copy read X + Y, two kernels concurrently", [&] {
        read_zc<8><<<sms * 2, 512, 0, s[0]>>>(n4, (const float4*)mx, dout);
        read_zc<8><<<sms * 2, 512, 0, s[1]>>>(n4, (const float4*)my, dout + 4);
    }, 2.0 * bytes);
    run("zero-copy write Y (D2H by SM stores), 4 blocks/SM",
        [&] { write_zc<<<sms * 4, 512, 0, s[0]>>>(n4, (float4*)my, (const float4*)dy); }, double(bytes));
    run("copy engine H2D X+Y  +  SM-store D2H of Y", [&] {
        cudaMemcpyAsync(dx, hx, bytes, cudaMemcpyHostToDevice, s[0]);
        cudaMemcpyAsync(dy, hy, bytes, cudaMemcpyHostToDevice, s[1]);
        write_zc<<<sms * 2, 512, 0, s[2]>>>(n4, (float4*)my, (const float4*)dx);
    }, mix);
    run("SM-load H2D X+Y  +  copy engine D2H of Y", [&] {
        read_zc<8><<<sms * 2, 512, 0, s[0]>>>(n4, (const float4*)mx, dout);
        read_zc<8><<<sms * 2, 512, 0, s[1]>>>(n4, (const float4*)my, dout + 4);
        cudaMemcpyAsync(hy, dy, bytes, cudaMemcpyDeviceToHost, s[2]);
    }, mix);
    return 0;
}
