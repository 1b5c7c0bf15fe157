// Probe: AXPY fp32 at n = 2^28 with bulk-copy (TMA) staging vs the production-style LDG.128
// streaming kernel. Bulk variant: persistent CTAs walk 16 KiB chunks of X and Y; one elected
// thread issues cp.async.bulk global->shared for both (mbarrier transaction count), the block
// computes y = a*x + y in shared memory, then cp.async.bulk shared->global writes Y back; a
// STAGES-deep ring overlaps loads of chunk c+1.. with the compute/store of chunk c.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("ERR %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int CHUNK_BYTES, int STAGES>
__global__ void __launch_bounds__(256) axpy_bulk(size_t n, float a, const float* __restrict__ x, float* __restrict__ y)
{
    extern __shared__ __align__(128) uint8_t sm[];
    constexpr int CF = CHUNK_BYTES / 4; // floats per chunk
    float* sx = reinterpret_cast<float*>(sm);
    float* sy = sx + STAGES * CF;
    uint64_t* full = reinterpret_cast<uint64_t*>(sy + STAGES * CF);
    const size_t nchunks = n / CF; // tail handled by the LDG kernel in a real integration
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](size_t c, int s) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&full[s])),
                     "r"(2 * CHUNK_BYTES) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                         smem_u32(sx + s * CF)), "l"(x + c * CF), "r"(CHUNK_BYTES), "r"(smem_u32(&full[s])) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                         smem_u32(sy + s * CF)), "l"(y + c * CF), "r"(CHUNK_BYTES), "r"(smem_u32(&full[s])) : "memory");
    };
    // chunks of this CTA: c = blockIdx.x + i * gridDim.x
    size_t c0 = blockIdx.x;
    if (threadIdx.x == 0)
        for (int s = 0; s < STAGES; ++s) {
            const size_t c = c0 + static_cast<size_t>(s) * gridDim.x;
            if (c < nchunks)
                issue(c, s);
        }
    int it = 0;
    for (size_t c = c0; c < nchunks; c += gridDim.x, ++it) {
        const int s = it % STAGES;
        const uint32_t parity = (it / STAGES) & 1;
        asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D_%=;\nbra W_%=;\nD_%=:\n}\n" ::"r"(
                         smem_u32(&full[s])), "r"(parity) : "memory");
        float4* vx = reinterpret_cast<float4*>(sx + s * CF);
        float4* vy = reinterpret_cast<float4*>(sy + s * CF);
        for (int i = threadIdx.x; i < CF / 4; i += blockDim.x) {
            const float4 xv = vx[i];
            float4 yv = vy[i];
            yv.x = __fadd_rn(__fmul_rn(a, xv.x), yv.x);
            yv.y = __fadd_rn(__fmul_rn(a, xv.y), yv.y);
            yv.z = __fadd_rn(__fmul_rn(a, xv.z), yv.z);
            yv.w = __fadd_rn(__fmul_rn(a, xv.w), yv.w);
            vy[i] = yv;
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(y + c * CF),
                         "r"(smem_u32(sy + s * CF)), "r"(CHUNK_BYTES) : "memory");
            asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
            // the slot is refilled only after its store has read the shared memory
            asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
            const size_t nc = c + static_cast<size_t>(STAGES) * gridDim.x;
            if (nc < nchunks)
                issue(nc, s);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0)
        asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

__global__ void __launch_bounds__(512) axpy_ldg(size_t n, float a, const float* __restrict__ x, float* __restrict__ y)
{
    const size_t i = (static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x);
    if (i * 4 + 3 < n) {
        const float4 xv = __ldcs(reinterpret_cast<const float4*>(x) + i);
        float4 yv = __ldcs(reinterpret_cast<const float4*>(y) + i);
        yv.x = __fadd_rn(__fmul_rn(a, xv.x), yv.x);
        yv.y = __fadd_rn(__fmul_rn(a, xv.y), yv.y);
        yv.z = __fadd_rn(__fmul_rn(a, xv.z), yv.z);
        yv.w = __fadd_rn(__fmul_rn(a, xv.w), yv.w);
        __stcs(reinterpret_cast<float4*>(y) + i, yv);
    }
}

template <class F>
float time_ms(F&& f, int reps)
{
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    f();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r)
        f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / reps;
}

template <int CHUNK, int STAGES>
int run_bulk(size_t n, float* x, float* y, int sms, int per_sm)
{
    const size_t smem = static_cast<size_t>(STAGES) * 2 * CHUNK + STAGES * 8;
    CK(cudaFuncSetAttribute(axpy_bulk<CHUNK, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    const float ms = time_ms([&] { axpy_bulk<CHUNK, STAGES><<<sms * per_sm, 256, smem>>>(n, 1.0000001f, x, y); }, 50);
    CK(cudaGetLastError());
    std::printf("bulk chunk=%6d B stages=%d ctas/SM=%d: %.4f ms  %.1f GB/s\n", CHUNK, STAGES, per_sm, ms, 12.0 * n / ms / 1e6);
    return 0;
}

int main()
{
    const size_t n = size_t(1) << 28;
    float *x, *y;
    CK(cudaMalloc(&x, n * 4));
    CK(cudaMalloc(&y, n * 4));
    cudaMemset(x, 0, n * 4);
    cudaMemset(y, 0, n * 4);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int r = 0; r < 2; ++r) {
        const float ms = time_ms([&] { axpy_ldg<<<static_cast<unsigned>(n / 4 / 512), 512>>>(n, 1.0000001f, x, y); }, 50);
        std::printf("ldg128 512 thr x 1 float4: %.4f ms  %.1f GB/s\n", ms, 12.0 * n / ms / 1e6);
        run_bulk<16384, 4>(n, x, y, sms, 1);
        run_bulk<16384, 4>(n, x, y, sms, 2);
        run_bulk<32768, 3>(n, x, y, sms, 1);
        run_bulk<8192, 6>(n, x, y, sms, 2);
        run_bulk<8192, 4>(n, x, y, sms, 3);
        run_bulk<4096, 8>(n, x, y, sms, 3);
    }
    // correctness spot check of the bulk kernel
    float* h = new float[1024];
    for (int i = 0; i < 1024; ++i) h[i] = float(i);
    cudaMemcpy(x, h, 4096, cudaMemcpyHostToDevice);
    cudaMemcpy(y, h, 4096, cudaMemcpyHostToDevice);
    axpy_bulk<16384, 4><<<sms, 256, 4 * 2 * 16384 + 32>>>(n, 2.0f, x, y);
    cudaMemcpy(h, y, 4096, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < 1024; ++i)
        bad += h[i] != 3.0f * float(i);
    std::printf("bulk correctness (first 1024): %d mismatches\n", bad);
    return 0;
}
