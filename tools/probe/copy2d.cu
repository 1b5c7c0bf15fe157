// Probe: pinned-host -> device cudaMemcpy2DAsync throughput vs row width (strided source),
// the cost model for staging sub-blocks of a host matrix (e2e DGEMM schedule).
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s @%d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)

int main()
{
    const size_t n = 8192, pitch = n * 8;
    double *h, *d;
    CK(cudaMallocHost(&h, n * pitch));
    CK(cudaMalloc(&d, n * pitch));
    for (size_t i = 0; i < n * n; i += 512) h[i] = double(i);
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (size_t w : {128, 256, 512, 1024, 2048, 4096, 8192}) {
        for (size_t rows : {512, 2048, 8192}) {
            const size_t bytes = w * 8 * rows;
            float best = 1e30f;
            for (int r = 0; r < 4; ++r) {
                cudaEventRecord(e0, s);
                // copy the sub-block [0,rows) x [0,w) into a dense w-wide device block
                CK(cudaMemcpy2DAsync(d, w * 8, h, pitch, w * 8, rows, cudaMemcpyHostToDevice, s));
                cudaEventRecord(e1, s);
                CK(cudaEventSynchronize(e1));
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                best = ms < best ? ms : best;
            }
            printf("H2D 2D width=%5zu cols (%6zu B rows) rows=%5zu: %8.3f ms  %6.1f GB/s\n", w, w * 8, rows, best,
                   bytes / best / 1e6);
        }
    }
    // D2H direction for the C write-back of a sub-block
    for (size_t w : {512, 2048, 8192}) {
        const size_t rows = 2048, bytes = w * 8 * rows;
        float best = 1e30f;
        for (int r = 0; r < 4; ++r) {
            cudaEventRecord(e0, s);
            CK(cudaMemcpy2DAsync(h, pitch, d, w * 8, w * 8, rows, cudaMemcpyDeviceToHost, s));
            cudaEventRecord(e1, s);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        printf("D2H 2D width=%5zu cols rows=%5zu: %8.3f ms  %6.1f GB/s\n", w, rows, best, bytes / best / 1e6);
    }
    return 0;
}
