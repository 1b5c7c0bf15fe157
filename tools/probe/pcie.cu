// PCIe probe: H2D with 1 vs 2 concurrent streams (copy engines), and H2D + D2H duplex.
#include <cstdio>
#include <cuda_runtime.h>
int main()
{
    const size_t bytes = size_t(512) << 20;
    char *h[3], *d[3];
    for (int i = 0; i < 3; ++i) {
        cudaMallocHost(&h[i], bytes);
        cudaMalloc(&d[i], bytes);
    }
    cudaStream_t s[3];
    for (auto& x : s)
        cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, auto&& body, double total) {
        body();
        cudaDeviceSynchronize();
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0, 0);
            cudaDeviceSynchronize();
            auto t = cudaEventRecord(e0, 0);
            (void)t;
            body();
            cudaDeviceSynchronize();
            cudaEventRecord(e1, 0);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        std::printf("%-34s %7.2f ms  %6.1f GB/s total\n", name, best, total / best / 1e6);
    };
    run("H2D 1 stream, 512 MB", [&] { cudaMemcpyAsync(d[0], h[0], bytes, cudaMemcpyHostToDevice, s[0]); }, bytes);
    run("H2D 2 streams, 2 x 512 MB", [&] {
        cudaMemcpyAsync(d[0], h[0], bytes, cudaMemcpyHostToDevice, s[0]);
        cudaMemcpyAsync(d[1], h[1], bytes, cudaMemcpyHostToDevice, s[1]);
    }, 2.0 * bytes);
    run("H2D 1 stream, 2 x 512 MB serial", [&] {
        cudaMemcpyAsync(d[0], h[0], bytes, cudaMemcpyHostToDevice, s[0]);
        cudaMemcpyAsync(d[1], h[1], bytes, cudaMemcpyHostToDevice, s[0]);
    }, 2.0 * bytes);
    run("D2H 1 stream, 512 MB", [&] { cudaMemcpyAsync(h[2], d[2], bytes, cudaMemcpyDeviceToHost, s[2]); }, bytes);
    run("H2D 2x512 + D2H 512 (AXPY mix)", [&] {
        cudaMemcpyAsync(d[0], h[0], bytes, cudaMemcpyHostToDevice, s[0]);
        cudaMemcpyAsync(d[1], h[1], bytes, cudaMemcpyHostToDevice, s[0]);
        cudaMemcpyAsync(h[2], d[2], bytes, cudaMemcpyDeviceToHost, s[2]);
    }, 3.0 * bytes);
    run("H2D 2 streams + D2H (AXPY mix)", [&] {
        cudaMemcpyAsync(d[0], h[0], bytes, cudaMemcpyHostToDevice, s[0]);
        cudaMemcpyAsync(d[1], h[1], bytes, cudaMemcpyHostToDevice, s[1]);
        cudaMemcpyAsync(h[2], d[2], bytes, cudaMemcpyDeviceToHost, s[2]);
    }, 3.0 * bytes);
    return 0;
}
