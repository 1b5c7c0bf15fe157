// DMMA throughput vs resident warps per SM and independent accumulators per warp.
#include <cstdio>
#include <cuda_runtime.h>
template <int ACC>
__global__ void dmma_k(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = threadIdx.x * 2e-3;
  double c[ACC][2];
#pragma unroll
  for (int i = 0; i < ACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5) out[0] = s;
}
template <int ACC> void run(double* out, int warps_per_sm) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int threads = warps_per_sm * 32 > 1024 ? 1024 : warps_per_sm * 32;
  int bps = warps_per_sm * 32 / threads;
  int blocks = 148 * bps; int iters = 4096 / ACC * 16;
  dmma_k<ACC><<<blocks, threads>>>(out, 10);
  cudaEventRecord(e0); dmma_k<ACC><<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
  cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * 256 * ACC * (double)iters * blocks * (threads / 32);
  printf("warps/SM=%2d acc/warp=%2d : %.2f TFLOP/s\n", warps_per_sm, ACC, fl / ms / 1e9);
}
int main() {
  double* out; cudaMalloc(&out, 8);
  for (int w : {4, 8, 12, 16}) { run<8>(out, w); run<16>(out, w); run<32>(out, w); }
  return 0;
}
