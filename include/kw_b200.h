/*
 * kw_b200.h — the C-ABI boundary of the B200-native kernelweave path (libkw_b200.so).
 *
 * The reference (kernelweave, /root/reference/proj) has exactly one compiled dispatch point
 * for kernels, `detail::runGrid(BackendKind, const WorkDiv&, const KernelBody&)`
 * (core/include/kernelweave/exec.hpp:23, core/src/accel.cpp:251-265). A host std::function
 * cannot run on a GPU, so this build replaces that seam — and the buffer / copy / queue
 * services the kernels are fed through — with the plain-pointer entry points below. The C++
 * drop-in headers (include/kernelweave/*.hpp) translate the reference's classes onto them;
 * INTEGRATION.md shows the ctypes / C++ bindings a maintainer adds.
 *
 * Conventions: no exceptions cross this boundary; every entry point returns a kw_status and
 * leaves a thread-local message in kw_last_error() on failure. Precondition violations are
 * reported before anything is enqueued (the reference's UsageError contract, e.g.
 * core/src/buffer.cpp:101-107, core/src/work_div.cpp:53-63). Index vectors are ordered
 * slowest-varying first with the LAST component fastest (index_vec.hpp:15-24); the last
 * component maps to CUDA x.
 *
 * There is no CPU fallback: every compute entry point runs a hand-written sm_100a kernel.
 */
#ifndef KW_B200_H
#define KW_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define KW_EXPORT __attribute__((visibility("default")))
#else
#define KW_EXPORT
#endif

/* Status codes. Mirrors the reference's error taxonomy (core/include/kernelweave/error.hpp):
 * KW_USAGE ~ UsageError (:13), KW_RESOURCE ~ ResourceError (:19), KW_TASK ~ TaskError (:26-40). */
typedef int kw_status;
#define KW_OK 0
#define KW_USAGE 1
#define KW_RESOURCE 2
#define KW_TASK 3

/* Queue flavours: QueueFlavor::Sync / ::Async (core/include/kernelweave/queue.hpp:21-24). */
#define KW_QUEUE_SYNC 0
#define KW_QUEUE_ASYNC 1

/* Task states: TaskState (queue.hpp:26-31). */
#define KW_TASK_PENDING 0
#define KW_TASK_RUNNING 1
#define KW_TASK_DONE 2
#define KW_TASK_FAILED 3

/* Memory kinds reported by kw_pointer_kind. */
#define KW_MEM_PAGEABLE 0 /* ordinary host memory unknown to CUDA */
#define KW_MEM_PINNED 1   /* page-locked host memory */
#define KW_MEM_DEVICE 2   /* device memory (any GPU) */

typedef struct kw_queue_s* kw_queue;
typedef struct kw_event_s* kw_event;

/* WorkDiv{blocksPerGrid, threadsPerBlock, elementsPerThread} (core/include/kernelweave/
 * work_div.hpp:33-53). `dim` in 1..3; unused trailing components must be 1. */
typedef struct {
    uint32_t dim;
    size_t blocks[3];
    size_t threads[3];
    size_t elems[3];
} kw_workdiv;

typedef struct {
    char name[96];
    int sm_count;
    int cc_major, cc_minor;
    size_t l2_bytes;
    size_t global_mem_bytes;
    size_t smem_per_block_optin;
    int sm_clock_khz;
    int mem_clock_khz;
    int mem_bus_width_bits;
} kw_device_props;

/* ---- errors ----------------------------------------------------------------------------- */
KW_EXPORT const char* kw_last_error(void);
KW_EXPORT const char* kw_version(void);

/* ---- devices (replaces Device::logical(i), core/include/kernelweave/device.hpp:14-37) ---- */
KW_EXPORT kw_status kw_device_count(int* n);
KW_EXPORT kw_status kw_device_props_get(int device, kw_device_props* props);
KW_EXPORT kw_status kw_device_synchronize(int device);
/* PCI bus id ("0000:1b:00.0" form, lower case) of a device: host code uses it to place pinned
 * staging buffers on the GPU's NUMA node (sysfs numa_node). */
KW_EXPORT kw_status kw_device_pci_bus_id(int device, char* buf, int len);

/* ---- buffers (replaces Buffer::Buffer / ~Buffer, core/src/buffer.cpp:25-46) --------------
 * device >= 0: device memory on that CUDA device; device == -1: page-locked host memory.
 * Pitch rule of buffer.cpp:37: 1-D dense; 2-D/3-D rows padded to row_align (power of two).
 * Returns the row pitch in bytes; storage = rowCount * pitch. */
KW_EXPORT kw_status kw_buffer_alloc(int device, uint32_t dim, const size_t extent[3], size_t elem_size,
                                    size_t row_align, void** ptr, size_t* row_pitch);
KW_EXPORT kw_status kw_buffer_free(int device, void* ptr);
KW_EXPORT kw_status kw_pointer_kind(const void* ptr, int* kind, int* device);
KW_EXPORT kw_status kw_memset(kw_queue q, void* ptr, int value, size_t bytes);

/* ---- queues (replaces Queue, queue.hpp:94-137 / core/src/queue.cpp) ----------------------
 * One CUDA stream per queue. Sync: every enqueue completes before returning. Async: enqueue
 * returns immediately. Launch failures are collected and surfaced by kw_queue_wait() as
 * KW_TASK with "task failed: <msg>" / "<n> tasks failed; first: <msg>" (error.hpp:26-40,
 * queue.cpp:108-131); the counters reset after a report. */
KW_EXPORT kw_status kw_queue_create(int device, int flavor, kw_queue* q);
KW_EXPORT kw_status kw_queue_destroy(kw_queue q);
KW_EXPORT kw_status kw_queue_wait(kw_queue q);
/* Sync queues only: the TaskError for failures since the last report, without a stream round
 * trip (every task on a Sync queue completed inside its own call; after a failure it drains the
 * stream first, like kw_queue_wait). What executeTask uses. KW_USAGE on an Async queue. */
KW_EXPORT kw_status kw_queue_report(kw_queue q);
KW_EXPORT kw_status kw_queue_device(kw_queue q, int* device);
KW_EXPORT kw_status kw_queue_flavor(kw_queue q, int* flavor);
KW_EXPORT kw_status kw_queue_stream(kw_queue q, void** cuda_stream);
KW_EXPORT kw_status kw_queue_shutdown(kw_queue q);

/* A kernel launch made OUTSIDE this library on q's stream (the header-only generic functor
 * launcher, include/kernelweave/cuda_exec.cuh) is one enqueue, bracketed by this pair:
 *   kw_queue_begin_launch  takes q's enqueue lock (FIFO order against every other enqueue on q),
 *                          rejects a shut-down queue (KW_USAGE, the reference's "enqueue on a
 *                          shut-down queue"), and returns q's stream and device plus a zeroed
 *                          device-side failure slot for the kernel (see kw_queue_fail_slot);
 *   kw_queue_end_launch    `cuda_error` = the launch's cudaGetLastError() value. Arms the slot
 *                          (only now can a drain of q resolve it), records a launch failure for
 *                          kw_queue_wait, counts the launch, completes the task on a Sync queue,
 *                          and releases the lock. Must follow every successful begin. */
KW_EXPORT kw_status kw_queue_begin_launch(kw_queue q, const char* what, void** cuda_stream, int* device,
                                          uint32_t** fail_slot);
KW_EXPORT kw_status kw_queue_end_launch(kw_queue q, int cuda_error, const char* what);

/* Legacy form of the pair above without the enqueue lock: kw_queue_fail_slot stages a slot for
 * the calling thread's next launch on q; kw_queue_complete_launch arms it and completes the
 * launch. Prefer begin/end (FIFO-safe against concurrent enqueues). */
KW_EXPORT kw_status kw_queue_complete_launch(kw_queue q, int cuda_error, const char* what);

/* Device-side task failure (the GPU form of "a kernel exception fails the task; later tasks
 * still run", queue.hpp:86-93 / accel.cpp:240-248): returns a zeroed 32-bit slot the NEXT launch
 * on q may set to a non-zero code from device code (kernelweave::failTask). The slot is
 * resolved when q's stream has drained (kw_queue_wait, or inside the enqueue of a Sync queue):
 * a non-zero code counts as one failed task, reported as `what: ... (code N)`. The next
 * kw_event_record on q attaches the slot to its event, whose state is then FAILED. */
KW_EXPORT kw_status kw_queue_fail_slot(kw_queue q, const char* what, uint32_t** slot);
/* Failure codes the library's own device code writes into a slot (user codes stay below). */
#define KW_FAIL_SHARED_OVERFLOW 0xFFFF0001u /* allocSharedMem beyond the block's shared memory */
#define KW_FAIL_READY_TIMEOUT 0xFFFF0002u   /* streamed DGEMM: a panel ready flag never arrived */

/* TaskHandle (queue.hpp:36-52) as a CUDA event recorded after the last enqueued task. State is
 * PENDING until the event completes, then DONE — or FAILED on a device fault or when the task's
 * device-side failure slot (kw_queue_fail_slot) was set. A task's own launch failure is the
 * KW_TASK returned by its kw_* call (the C++/Python handles carry it; a Sync queue's handles need
 * no event at all). */
KW_EXPORT kw_status kw_event_record(kw_queue q, kw_event* ev);
/* The same completion marker without a timestamp (cheaper to record and to wait on): what the
 * C++ and Python TaskHandles of an Async queue use. kw_event_elapsed_ms rejects it. */
KW_EXPORT kw_status kw_task_marker(kw_queue q, kw_event* ev);
KW_EXPORT kw_status kw_event_state(kw_event ev, int* state);
KW_EXPORT kw_status kw_event_destroy(kw_event ev);
/* Milliseconds between two recorded events of the same device (timing helper). */
KW_EXPORT kw_status kw_event_elapsed_ms(kw_event start, kw_event stop, float* ms);

/* ---- copies (replaces createCopy/copyBuffer, core/src/buffer.cpp:99-151) -----------------
 * Deep copy of `extent` elements from the origin corner of src to the origin corner of dst.
 * Each side's rows are located via its own extent and pitch; bytes outside the copied box
 * are never touched. Any combination of host / pinned / device memory (UVA). */
KW_EXPORT kw_status kw_copy(kw_queue q, void* dst, size_t dst_pitch, const size_t dst_extent[3],
                            const void* src, size_t src_pitch, const size_t src_extent[3], uint32_t dim,
                            const size_t extent[3], size_t elem_size);

/* ---- work division helpers (work_div.cpp:65-119) ---------------------------------------- */
/* totalExtent(wd, origin, unit); origin 0 Grid,1 Block,2 Thread; unit 0 Blocks,1 Threads,2 Elems */
KW_EXPORT kw_status kw_total_extent(const kw_workdiv* wd, int origin, int unit, size_t out[3]);
/* divideForBackend for the GPU: thread-level shape ceil(N/(B*V)) x B x V (work_div.cpp:96-119). */
KW_EXPORT kw_status kw_divide_for_gpu(uint32_t dim, const size_t problem[3], const size_t threads_hint[3],
                                      const size_t elems_hint[3], kw_workdiv* out);
/* The library's preferred division for each kernel (NULL wd in the calls below uses it). */
KW_EXPORT kw_status kw_axpy_default_workdiv(size_t n, int elem_size, kw_workdiv* out);
KW_EXPORT kw_status kw_dgemm_default_workdiv(size_t m, size_t n, size_t tile, kw_workdiv* out);

/* ---- K1: AXPY  Y = alpha*X + Y  (AxpyKernel, core/src/kernels/axpy.cpp:10-23) ------------
 * Bit-exact against axpyReference (reference.cpp:8-12): product and sum rounded separately
 * (no FMA contraction). wd covers n with its grid element extent; elements >= n are never
 * touched (axpy.cpp:15-17). Device pointers run the HBM kernel; host pointers (pinned or
 * pageable) are streamed through the device in 32 MiB chunks, uploads / kernel / downloads
 * overlapped on three streams (e2e path). wd == NULL: kw_axpy_default_workdiv. */
KW_EXPORT kw_status kw_axpy_f32(kw_queue q, const kw_workdiv* wd, size_t n, float alpha, const float* x,
                                float* y);
KW_EXPORT kw_status kw_axpy_f64(kw_queue q, const kw_workdiv* wd, size_t n, double alpha, const double* x,
                                double* y);
/* Name of the kernel template a device-resident kw_axpy_* launch with this division runs for
 * these operand addresses (alignment decides the vector path; nothing is dereferenced). */
KW_EXPORT kw_status kw_axpy_kernel_name(const kw_workdiv* wd, int elem_size, const void* x, const void* y,
                                        char* buf, size_t len);

/* ---- K2: tiled DGEMM  C = alpha*A*B + beta*C  (GemmTiledKernel, gemm.cpp:40-118) ----------
 * Row-major pitched fp64; lda/ldb/ldc in elements. FP64 DMMA tensor-core kernel fed by TMA and
 * an mbarrier stage ring (warp-specialised; a cp.async kernel for operands TMA cannot address).
 * Within |dC| <= (K+4)*2^-53*|C_ref| of gemmReference (reference.cpp:14-26); the epilogue is
 * fl(fl(alpha*acc) + fl(beta*c)) as in gemm.cpp:115. beta multiplies C even when 0 (C is always
 * read). wd == NULL: default tile; wd's tile (64 or 128) is the coverage contract, the CTA tile is
 * chosen per problem among bitwise-identical configurations. Host pointers are streamed through
 * the device inside the task (row panels, or for compute-heavy problems with all three operands
 * pinned, panel uploads feeding one persistent launch); bits equal the resident launch.
 * Environment KW_DGEMM_SPLITK=1 (read once) opts into split-k (config 27) for fewer 32x32 output
 * tiles than SMs with k >= 1024: faster there, within the same bound, deterministic, but not
 * bitwise equal to the host-streamed / row-sharded paths for those shapes. */
KW_EXPORT kw_status kw_dgemm(kw_queue q, const kw_workdiv* wd, size_t m, size_t n, size_t k, double alpha,
                             const double* A, size_t lda, const double* B, size_t ldb, double beta, double* C,
                             size_t ldc);

/* K2 bitwise mode: the tiled DGEMM with separately rounded products and sums in ascending k —
 * BITWISE equal to gemmReference and to the reference's GemmTiledKernel (test_kernels.cpp:208-230
 * pins tiled == naive bitwise). FP64 pipe bound (two operations per term). 128x128 tiles of 256
 * threads; device operands. */
KW_EXPORT kw_status kw_dgemm_bitwise(kw_queue q, const kw_workdiv* wd, size_t m, size_t n, size_t k, double alpha,
                                     const double* A, size_t lda, const double* B, size_t ldb, double beta, double* C,
                                     size_t ldc);

/* Tile-configuration sweep (BASELINE.json configs[4]): the DMMA kernel's instantiated
 * configurations, info = {BM, BN, BK, threads, stages}; device operands only. Configurations
 * 14..26, 28, 29 are bitwise interchangeable; 27 is split-k (sums of k-slice chains, see kw_dgemm). */
KW_EXPORT int kw_dgemm_config_count(void);
KW_EXPORT kw_status kw_dgemm_config_info(int cfg, int info[5]);
KW_EXPORT kw_status kw_dgemm_with_config(kw_queue q, int cfg, size_t m, size_t n, size_t k, double alpha,
                                         const double* A, size_t lda, const double* B, size_t ldb, double beta,
                                         double* C, size_t ldc);

/* ---- K3: naive DGEMM (GemmNaiveKernel, gemm.cpp:11-38) — BIT-EXACT mode --------------------
 * One dot product per output, ascending p, products and sums rounded separately, acc from
 * +0.0: bitwise identical to gemmReference. Computes exactly the outputs the (rows, cols) work
 * division covers in the reference (thread (r, c) owns rows [r*er, r*er+er) x cols [c*ec, ...));
 * inside a block the outputs go to lanes in column order (coalesced; no bit depends on it). */
KW_EXPORT kw_status kw_dgemm_naive(kw_queue q, const kw_workdiv* wd, size_t m, size_t n, size_t k,
                                   double alpha, const double* A, size_t lda, const double* B, size_t ldb,
                                   double beta, double* C, size_t ldc);

/* ---- multi-GPU (one process per GPU; BASELINE.json configs[3]) ------------------
 * NCCL communicator for the row-sharded DGEMM's broadcast of B. The 128-byte unique id is
 * produced by rank 0 (kw_comm_unique_id) and exchanged by the caller (torch.distributed
 * store, MPI, a file). */
typedef struct kw_comm_s* kw_comm;
KW_EXPORT kw_status kw_comm_unique_id(unsigned char id[128]);
KW_EXPORT kw_status kw_comm_init(kw_comm* comm, int device, int world, int rank, const unsigned char id[128]);
KW_EXPORT kw_status kw_comm_destroy(kw_comm comm);
KW_EXPORT kw_status kw_comm_broadcast(kw_comm comm, kw_queue q, void* buf, size_t bytes, int root);

/* Row-block shard of C = alpha*A*B + beta*C across `world` ranks: this rank holds
 * rows [row0, row0+m_local) of A (lda) and C (ldc); B (k x n, ldb) is valid on `root` and is
 * broadcast in `panels` column panels into the caller's b_panels scratch
 * (kw_dgemm_rowsharded_scratch doubles, panel-major: panel j is k x w_j with leading dimension
 * w_j rounded up to 8 — the Buffer pitch rule, so every panel is TMA-addressable), each panel's
 * broadcast (high-priority stream; every rank, world 1 included, runs ncclBroadcast) overlapped
 * with the DGEMMs of earlier panels, which alternate between two compute streams.
 * Every output element is reduced entirely on
 * one rank in the single-GPU kernel's order, so the gathered C is bitwise identical to the
 * 1-GPU kw_dgemm result. */
KW_EXPORT kw_status kw_dgemm_rowsharded(kw_comm comm, kw_queue q, size_t m_local, size_t n, size_t k,
                                        double alpha, const double* A, size_t lda, const double* B, size_t ldb,
                                        double beta, double* C, size_t ldc, double* b_panels, int panels,
                                        int root);
/* Doubles the b_panels scratch of kw_dgemm_rowsharded must hold for (n, k, panels). */
KW_EXPORT kw_status kw_dgemm_rowsharded_scratch(size_t n, size_t k, int panels, size_t* elems);

/* SPLIT DGEMM schedule of CTA `cta` of `ctas` (host-side view of the device planner, for tests):
 * out = {ndp, dp0, dp_step, head, nfull, tail, t_head, x_head, t_full0, t_tail, x_tail};
 * dp_tiles < 0 = the library's default data-parallel share. */
KW_EXPORT kw_status kw_dgemm_split_plan(long long tiles, long long ktiles, long long ctas, long long cta,
                                        long long dp_tiles, int out[11]);

/* Measurement: SPLIT DGEMM launches after this call stamp their timeline into `device_buffer`
 * (40 u64 per virtual CTA: %globaltimer at start, SM id, start/end of up to 18 pieces, end);
 * NULL turns it off. Only a library compiled with -DKW_SPLIT_TRACE stamps (a no-op otherwise). */
KW_EXPORT kw_status kw_dgemm_split_trace(void* device_buffer);

/* ---- measurement helpers (bench / tests) --------------------------------------------------- */
/* Writes a device scratch buffer larger than L2 (flush between timed iterations). */
KW_EXPORT kw_status kw_l2_flush(kw_queue q);
/* Number of kernels this library launched in the process so far (gpu_launches claim). */
KW_EXPORT uint64_t kw_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* KW_B200_H */
