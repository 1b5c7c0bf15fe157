// Hardware probe: FP64 DFMA vs DMMA peak, simple AXPY bandwidth, device props.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s @%d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)

__global__ void dfma_peak(double* out, int iters, double a, double b) {
  double c[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 1234.5) out[0] = s;
}

__global__ void dmma_peak(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = threadIdx.x * 2e-3;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5) out[0] = s;
}

__global__ void axpy_f4(size_t n4, float alpha, const float4* __restrict__ x, float4* __restrict__ y) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 xv = x[i], yv = y[i];
    yv.x = __fadd_rn(__fmul_rn(alpha, xv.x), yv.x);
    yv.y = __fadd_rn(__fmul_rn(alpha, xv.y), yv.y);
    yv.z = __fadd_rn(__fmul_rn(alpha, xv.z), yv.z);
    yv.w = __fadd_rn(__fmul_rn(alpha, xv.w), yv.w);
    y[i] = yv;
  }
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("name=%s sms=%d l2=%d smemPerBlockOptin=%zu regsPerSM=%d clockKHz=%d memClockKHz=%d busWidth=%d\n",
         p.name, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerBlockOptin, p.regsPerMultiprocessor,
         p.clockRate, p.memoryClockRate, p.memoryBusWidth);
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int bpsm : {4, 8}) {
    int iters = 20000; int threads = 256; int blocks = sms * bpsm;
    dfma_peak<<<blocks, threads>>>(out, 100, 1.0000001, 1e-9);
    cudaEventRecord(e0); dfma_peak<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * iters * (double)blocks * threads;
    printf("DFMA blocks/SM=%d: %.3f ms  %.2f TFLOP/s\n", bpsm, ms, fl / ms / 1e9);
  }
  for (int bpsm : {2, 4, 8}) {
    int iters = 20000; int threads = 256; int blocks = sms * bpsm;
    dmma_peak<<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0); dmma_peak<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 256 * 8 * iters * (double)blocks * (threads / 32);
    printf("DMMA m8n8k4 blocks/SM=%d: %.3f ms  %.2f TFLOP/s\n", bpsm, ms, fl / ms / 1e9);
  }
  size_t n = 1ull << 28;
  float *x, *y; CK(cudaMalloc(&x, n * 4)); CK(cudaMalloc(&y, n * 4));
  cudaMemset(x, 0, n * 4); cudaMemset(y, 0, n * 4);
  for (int threads : {256, 512}) for (int bpsm : {4, 8, 16, 64}) {
    int blocks = sms * bpsm * 256 / threads; if (bpsm == 64) blocks = (int)((n / 4 + threads - 1) / threads);
    axpy_f4<<<blocks, threads>>>(n / 4, 1.5f, (float4*)x, (float4*)y);
    float best = 1e9;
    for (int r = 0; r < 10; ++r) {
      cudaEventRecord(e0); axpy_f4<<<blocks, threads>>>(n / 4, 1.5f, (float4*)x, (float4*)y); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("AXPY f32 2^28 threads=%d blocks=%d: %.4f ms  %.1f GB/s\n", threads, blocks, best, 12.0 * n / best / 1e6);
  }
  return 0;
}
