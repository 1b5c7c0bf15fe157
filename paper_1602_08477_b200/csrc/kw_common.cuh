// kw_common.cuh — shared plumbing of libkw_b200.so: status/error reporting across the C-ABI,
// the queue object (a CUDA stream standing in for kernelweave's Queue, queue.hpp:94-137) and
// the launch bookkeeping every kernel entry point goes through.
#pragma once

#include "kw_b200.h"

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <atomic>
#include <cstdio>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

namespace kw {

// Thread-local message behind kw_last_error().
void set_error(const std::string& msg);
const std::string& last_error();

// Number of kernels launched by this library (the bench's gpu_launches claim).
extern std::atomic<uint64_t> g_launches;

// A device-side failure slot of one launch (kw_queue_fail_slot): mapped pinned memory the
// kernel may write; resolved (copied to `code`, slot recycled) once the queue's stream drained.
struct FailSlot {
    std::mutex mu;
    uint32_t* slot = nullptr; // nullptr once resolved
    uint32_t code = 0;
    std::string what;
    uint32_t read()
    {
        std::lock_guard<std::mutex> lock(mu);
        return slot ? *reinterpret_cast<volatile uint32_t*>(slot) : code;
    }
};

struct Queue {
    int device = 0;
    int flavor = KW_QUEUE_SYNC;
    cudaStream_t stream = nullptr; // in-order FIFO of the queue
    cudaStream_t aux = nullptr;    // D2H stream of the host-staged paths
    cudaStream_t h2d = nullptr;    // H2D stream of the host-staged paths
    cudaStream_t comp2 = nullptr;  // second compute stream (panel launches overlap their tails)
    std::mutex mu;       // failure bookkeeping
    std::mutex enqueue;  // serialises enqueues from several host threads (queue.hpp:89-93)
    size_t failed = 0;
    std::string first_failure;
    bool shut = false;
    // Device scratch for host-staged execution (grown on demand, freed with the queue).
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
    static constexpr int kRing = 4;
    cudaEvent_t ev_ready[kRing] = {};  // chunk computed -> D2H may start
    cudaEvent_t ev_free[kRing] = {};   // chunk drained  -> slot reusable
    cudaEvent_t ev_h2d[kRing] = {};    // chunk uploaded -> compute may start
    cudaEvent_t ev_join = nullptr;
    cudaEvent_t ev_join2 = nullptr;
    cudaEvent_t ev_start = nullptr;
    cudaEvent_t ev_b = nullptr;
    static constexpr int kBPanels = 8;
    cudaEvent_t ev_bp[kBPanels] = {}; // B column panel j uploaded (DGEMM e2e streaming)
    // Streamed e2e DGEMM: the tile order (pinned host copy + device copy), the key it was built
    // for and the event of its last upload.
    void* order_host = nullptr;
    void* order_dev = nullptr;
    size_t order_bytes = 0;
    size_t order_key[8] = {};
    cudaEvent_t ev_order = nullptr;
    // Device-side failure slots of launches not yet resolved (guarded by mu), and the slot the
    // next kw_event_record attaches to its event.
    // A slot joins pending_slots only once its kernel is in the stream (armed by
    // kw_queue_end_launch / kw_queue_complete_launch): a drain that began before the launch
    // must not resolve (and recycle) it.
    std::vector<std::shared_ptr<FailSlot>> pending_slots;
    std::shared_ptr<FailSlot> last_slot;
    std::shared_ptr<FailSlot> staged; // kw_queue_begin_launch .. end_launch (enqueue lock held)
};

// RAII device selector: the reference's queues are bound to one device; every entry point
// makes that device current for its duration. cudaSetDevice runs even when the device number
// already matches: it also makes the device's primary context current on a host thread that has
// not touched CUDA yet, which the driver-API calls behind the runtime (cuTensorMapEncodeTiled,
// cuStreamWriteValue32) need — without it a first call from a new thread silently fell back from
// the TMA kernel to the cp.async one (other bits, lower rate).
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev)
    {
        cudaGetDevice(&prev);
        cudaSetDevice(dev);
    }
    ~DeviceGuard()
    {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev)
            cudaSetDevice(prev);
    }
};

kw_status usage(const std::string& msg);
kw_status resource(const std::string& msg);
kw_status cuda_fail(const char* what, cudaError_t e);

// Records a failed task on the queue (reported by the next kw_queue_wait) and returns KW_TASK.
kw_status task_fail(Queue* q, const std::string& msg);

// After enqueuing one task: surfaces launch errors into the queue's failure list and, for a
// Sync queue, completes the task before returning (queue.cpp:21-23, 57-72).
kw_status after_enqueue(Queue* q, const char* what);

// Device-side failure slots are resolved in two steps around a drain of q->stream: take the
// armed slots (their kernels are already in the stream) BEFORE synchronising, then read, count
// (if `count_failures`) and recycle exactly those once the stream has drained.
std::vector<std::shared_ptr<FailSlot>> take_slots(Queue* q);
kw_status resolve_slots(Queue* q, std::vector<std::shared_ptr<FailSlot>>& slots, bool count_failures);

// A fresh zeroed mapped slot (nullptr when pinned allocation fails) / its release.
std::shared_ptr<FailSlot> make_slot(const std::string& what);
void release_slot(FailSlot& fs);
// Makes a slot whose writer is already enqueued on q->stream pending (and the next event's slot).
void arm_slot(Queue* q, std::shared_ptr<FailSlot> fs);

// SPLIT DGEMM launches keep per-stream scratch (kw_dgemm.cu): the abort word a bounded piece
// wait sets (read and cleared here by kw_queue_wait), and the release on queue destruction.
uint32_t split_take_abort(cudaStream_t s);
void split_release(cudaStream_t s);

// Ensures q->scratch holds at least `bytes` of device memory on q's device.
kw_status ensure_scratch(Queue* q, size_t bytes);

// Classifies a pointer: KW_MEM_PAGEABLE / KW_MEM_PINNED / KW_MEM_DEVICE.
int pointer_kind(const void* p, int* device);

inline size_t ceil_div(size_t a, size_t b) { return (a + b - 1) / b; }

// NVTX range around one library call (Nsight Systems timelines; header-only NVTX3, a no-op
// unless a tool is attached) — the tracing hook SURVEY.md §2 lists for the B200 build.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

} // namespace kw

#define KW_CHECK_QUEUE(q)                                                                          \
    do {                                                                                           \
        if ((q) == nullptr)                                                                        \
            return kw::usage("null queue");                                                        \
        if (reinterpret_cast<kw::Queue*>(q)->shut)                                                 \
            return kw::usage("queue: enqueue after shutdown");                                     \
    } while (0)

// Enqueue entry points hold the queue's enqueue lock for their whole body: arrival order at the
// lock is the FIFO order, and the host-staging scratch/events of one queue are never shared by
// two in-flight enqueues.
#define KW_ENQUEUE_LOCK(q) std::lock_guard<std::mutex> kw_enqueue_guard_(reinterpret_cast<kw::Queue*>(q)->enqueue)
#define KW_NVTX(name) kw::NvtxRange kw_nvtx_range_(name)
