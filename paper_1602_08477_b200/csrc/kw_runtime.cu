// kw_runtime.cu — devices, pitched buffers, queues (CUDA streams), task events, pitched copies
// and work-division arithmetic behind the C-ABI in include/kw_b200.h.
//
// Reference semantics followed here (paths relative to /root/reference/proj):
//   Buffer pitch rule / allocation errors      core/src/buffer.cpp:25-46
//   createCopy validation + per-row copy       core/src/buffer.cpp:99-146
//   Queue Sync/Async + failure collection      core/src/queue.cpp:21-131, queue.hpp:86-137
//   totalExtent / divideForBackend             core/src/work_div.cpp:53-119
#include "kw_common.cuh"

#include <cstdint>

#include <cctype>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

namespace kw {

static thread_local std::string t_error;
std::atomic<uint64_t> g_launches{0};

void set_error(const std::string& msg) { t_error = msg; }
const std::string& last_error() { return t_error; }

kw_status usage(const std::string& msg)
{
    set_error(msg);
    return KW_USAGE;
}

kw_status resource(const std::string& msg)
{
    set_error(msg);
    return KW_RESOURCE;
}

kw_status cuda_fail(const char* what, cudaError_t e)
{
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    cudaGetLastError(); // reported here: must not resurface as the next task's launch error
    return KW_TASK;
}

kw_status task_fail(Queue* q, const std::string& msg)
{
    cudaGetLastError(); // recorded once here (a device fault stays sticky regardless)
    {
        std::lock_guard<std::mutex> lock(q->mu);
        if (q->failed++ == 0)
            q->first_failure = msg;
    }
    set_error(msg);
    return KW_TASK;
}

namespace {
std::mutex g_slot_mu;
std::vector<uint32_t*> g_free_slots; // mapped pinned pages carved into 32-bit slots

uint32_t* slot_alloc()
{
    std::lock_guard<std::mutex> lock(g_slot_mu);
    if (g_free_slots.empty()) {
        constexpr size_t kSlots = 4096;
        void* page = nullptr;
        if (cudaHostAlloc(&page, kSlots * sizeof(uint32_t), cudaHostAllocMapped | cudaHostAllocPortable) !=
            cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        for (size_t i = 0; i < kSlots; ++i)
            g_free_slots.push_back(static_cast<uint32_t*>(page) + i);
    }
    uint32_t* s = g_free_slots.back();
    g_free_slots.pop_back();
    *reinterpret_cast<volatile uint32_t*>(s) = 0;
    return s;
}

void slot_release(uint32_t* s)
{
    std::lock_guard<std::mutex> lock(g_slot_mu);
    g_free_slots.push_back(s);
}
} // namespace

std::shared_ptr<FailSlot> make_slot(const std::string& what)
{
    auto fs = std::make_shared<FailSlot>();
    fs->slot = slot_alloc();
    if (!fs->slot)
        return nullptr;
    fs->what = what;
    return fs;
}

void release_slot(FailSlot& fs)
{
    std::lock_guard<std::mutex> lock(fs.mu);
    if (fs.slot) {
        fs.code = *reinterpret_cast<volatile uint32_t*>(fs.slot);
        slot_release(fs.slot);
        fs.slot = nullptr;
    }
}

void arm_slot(Queue* q, std::shared_ptr<FailSlot> fs)
{
    std::lock_guard<std::mutex> lock(q->mu);
    q->pending_slots.push_back(fs);
    q->last_slot = std::move(fs);
}

std::vector<std::shared_ptr<FailSlot>> take_slots(Queue* q)
{
    std::vector<std::shared_ptr<FailSlot>> out;
    std::lock_guard<std::mutex> lock(q->mu);
    out.swap(q->pending_slots);
    return out;
}

namespace {
// Failure codes the runtime itself writes from device code (kw_b200.h KW_FAIL_*).
std::string failure_text(const FailSlot& fs, uint32_t code)
{
    switch (code) {
    case KW_FAIL_SHARED_OVERFLOW:
        return fs.what + ": allocSharedMem request exceeds the block's shared memory (the reference's UsageError, "
                         "accel.cpp:286-292)";
    case KW_FAIL_READY_TIMEOUT:
        return fs.what + ": a streamed operand panel was never published (ready-flag wait timed out)";
    default:
        return fs.what + ": device functor reported failure (code " + std::to_string(code) + ")";
    }
}
} // namespace

kw_status resolve_slots(Queue* q, std::vector<std::shared_ptr<FailSlot>>& slots, bool count_failures)
{
    kw_status st = KW_OK;
    for (auto& fs : slots) {
        release_slot(*fs);
        if (fs->code != 0 && count_failures)
            st = task_fail(q, failure_text(*fs, fs->code));
    }
    slots.clear();
    return st;
}

kw_status after_enqueue(Queue* q, const char* what)
{
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        return task_fail(q, std::string(what) + ": " + cudaGetErrorString(e));
    if (q->flavor == KW_QUEUE_SYNC) {
        auto slots = take_slots(q);
        e = cudaStreamSynchronize(q->stream);
        if (e != cudaSuccess) {
            resolve_slots(q, slots, false);
            return task_fail(q, std::string(what) + ": " + cudaGetErrorString(e));
        }
        return resolve_slots(q, slots, true);
    }
    return KW_OK;
}

kw_status ensure_scratch(Queue* q, size_t bytes)
{
    if (q->scratch_bytes >= bytes)
        return KW_OK;
    DeviceGuard g(q->device);
    if (q->scratch) {
        cudaStreamSynchronize(q->stream);
        cudaStreamSynchronize(q->aux);
        cudaStreamSynchronize(q->h2d);
        cudaStreamSynchronize(q->comp2);
        cudaFree(q->scratch);
        q->scratch = nullptr;
        q->scratch_bytes = 0;
    }
    cudaError_t e = cudaMalloc(&q->scratch, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return resource("queue scratch: allocation of " + std::to_string(bytes) + " bytes failed");
    }
    q->scratch_bytes = bytes;
    return KW_OK;
}

int pointer_kind(const void* p, int* device)
{
    cudaPointerAttributes a;
    if (device)
        *device = -1;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return KW_MEM_PAGEABLE;
    }
    if (device)
        *device = a.device;
    switch (a.type) {
    case cudaMemoryTypeDevice:
    case cudaMemoryTypeManaged:
        return KW_MEM_DEVICE;
    case cudaMemoryTypeHost:
        return KW_MEM_PINNED;
    default:
        return KW_MEM_PAGEABLE;
    }
}

} // namespace kw

using kw::Queue;

struct kw_event_s {
    int device;
    cudaEvent_t ev;
    Queue* q;
    std::shared_ptr<kw::FailSlot> slot; // device-side failure slot of the task, if any
    bool timing = true;                 // false: kw_task_marker (no timestamp)
};

extern "C" {

const char* kw_last_error(void) { return kw::last_error().c_str(); }

const char* kw_version(void) { return "kw_b200 0.1 (sm_100a)"; }

kw_status kw_device_count(int* n)
{
    if (!n)
        return kw::usage("kw_device_count: null output");
    cudaError_t e = cudaGetDeviceCount(n);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *n = 0;
        return kw::cuda_fail("cudaGetDeviceCount", e);
    }
    return KW_OK;
}

kw_status kw_device_props_get(int device, kw_device_props* props)
{
    if (!props)
        return kw::usage("kw_device_props_get: null output");
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || device < 0 || device >= count) {
        cudaGetLastError();
        return kw::usage("kw_device_props_get: device index " + std::to_string(device) + " does not exist");
    }
    cudaDeviceProp p;
    cudaError_t e = cudaGetDeviceProperties(&p, device);
    if (e != cudaSuccess)
        return kw::cuda_fail("cudaGetDeviceProperties", e);
    std::memset(props, 0, sizeof(*props));
    std::strncpy(props->name, p.name, sizeof(props->name) - 1);
    props->sm_count = p.multiProcessorCount;
    props->cc_major = p.major;
    props->cc_minor = p.minor;
    props->l2_bytes = static_cast<size_t>(p.l2CacheSize);
    props->global_mem_bytes = p.totalGlobalMem;
    props->smem_per_block_optin = p.sharedMemPerBlockOptin;
    int clk = 0, mclk = 0, bus = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, device);
    cudaDeviceGetAttribute(&mclk, cudaDevAttrMemoryClockRate, device);
    cudaDeviceGetAttribute(&bus, cudaDevAttrGlobalMemoryBusWidth, device);
    props->sm_clock_khz = clk;
    props->mem_clock_khz = mclk;
    props->mem_bus_width_bits = bus;
    return KW_OK;
}

kw_status kw_device_pci_bus_id(int device, char* buf, int len)
{
    if (!buf || len < 13)
        return kw::usage("kw_device_pci_bus_id: buffer must hold at least 13 bytes");
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || device < 0 || device >= count) {
        cudaGetLastError();
        return kw::usage("kw_device_pci_bus_id: device index " + std::to_string(device) + " does not exist");
    }
    char id[64] = {};
    cudaError_t e = cudaDeviceGetPCIBusId(id, sizeof(id), device);
    if (e != cudaSuccess)
        return kw::cuda_fail("cudaDeviceGetPCIBusId", e);
    // CUDA reports "0000:1B:00.0" (possibly with an 8-digit domain); sysfs uses 4 lower-case digits.
    std::string s(id);
    const size_t colon = s.find(':');
    if (colon != std::string::npos && colon > 4)
        s = s.substr(colon - 4);
    for (char& ch : s)
        ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
    std::snprintf(buf, static_cast<size_t>(len), "%s", s.c_str());
    return KW_OK;
}

kw_status kw_device_synchronize(int device)
{
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || device < 0 || device >= count) {
        cudaGetLastError();
        return kw::usage("kw_device_synchronize: device index " + std::to_string(device) + " does not exist");
    }
    kw::DeviceGuard g(device);
    cudaError_t e = cudaDeviceSynchronize();
    return e == cudaSuccess ? KW_OK : kw::cuda_fail("cudaDeviceSynchronize", e);
}

// ---- buffers ------------------------------------------------------------------------------

kw_status kw_buffer_alloc(int device, uint32_t dim, const size_t extent[3], size_t elem_size, size_t row_align,
                          void** ptr, size_t* row_pitch)
{
    if (!ptr || !row_pitch || !extent)
        return kw::usage("Buffer: null argument");
    if (dim < 1 || dim > 3)
        return kw::usage("IndexVec: dimensionality must be 1, 2 or 3");
    if (elem_size == 0)
        return kw::usage("Buffer: element size must be positive");
    if (row_align == 0 || (row_align & (row_align - 1)) != 0 || row_align > (SIZE_MAX >> 2))
        return kw::usage("Buffer: row alignment must be a power of two");
    size_t rows = 1;
    for (uint32_t k = 0; k < dim; ++k) {
        if (extent[k] == 0)
            return kw::usage("Buffer: extent components must be positive");
        if (k + 1 < dim && __builtin_mul_overflow(rows, extent[k], &rows))
            return kw::resource("Buffer: size overflows the address space");
    }
    size_t row_bytes = 0, bytes = 0;
    if (__builtin_mul_overflow(extent[dim - 1], elem_size, &row_bytes) || row_bytes > (SIZE_MAX >> 1))
        return kw::resource("Buffer: size overflows the address space");
    // 1-D buffers are dense; padding a vector has no locality benefit (buffer.cpp:36-37).
    const size_t pitch = dim == 1 ? row_bytes : (row_bytes + row_align - 1) / row_align * row_align;
    if (__builtin_mul_overflow(rows, pitch, &bytes))
        return kw::resource("Buffer: size overflows the address space");
    void* p = nullptr;
    cudaError_t e;
    if (device < 0) {
        e = cudaMallocHost(&p, bytes);
    }
    else {
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || device >= count) {
            cudaGetLastError();
            return kw::usage("Buffer: device index " + std::to_string(device) + " does not exist");
        }
        kw::DeviceGuard g(device);
        e = cudaMalloc(&p, bytes);
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        return kw::resource("Buffer: allocation of " + std::to_string(bytes) + " bytes failed");
    }
    *ptr = p;
    *row_pitch = pitch;
    return KW_OK;
}

kw_status kw_buffer_free(int device, void* ptr)
{
    if (!ptr)
        return KW_OK;
    cudaError_t e;
    if (device < 0) {
        e = cudaFreeHost(ptr);
    }
    else {
        kw::DeviceGuard g(device);
        e = cudaFree(ptr);
    }
    return e == cudaSuccess ? KW_OK : kw::cuda_fail("Buffer free", e);
}

kw_status kw_pointer_kind(const void* ptr, int* kind, int* device)
{
    if (!kind)
        return kw::usage("kw_pointer_kind: null output");
    *kind = kw::pointer_kind(ptr, device);
    return KW_OK;
}

kw_status kw_memset(kw_queue qh, void* ptr, int value, size_t bytes)
{
    KW_CHECK_QUEUE(qh);
    KW_ENQUEUE_LOCK(qh);
    auto* q = reinterpret_cast<Queue*>(qh);
    kw::DeviceGuard g(q->device);
    cudaError_t e = cudaMemsetAsync(ptr, value, bytes, q->stream);
    if (e != cudaSuccess)
        return kw::task_fail(q, std::string("memset: ") + cudaGetErrorString(e));
    return kw::after_enqueue(q, "memset");
}

// ---- queues -------------------------------------------------------------------------------

kw_status kw_queue_create(int device, int flavor, kw_queue* out)
{
    if (!out)
        return kw::usage("Queue: null output");
    if (flavor != KW_QUEUE_SYNC && flavor != KW_QUEUE_ASYNC)
        return kw::usage("Queue: unknown flavor");
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || device < 0 || device >= count) {
        cudaGetLastError();
        return kw::usage("Queue: device index " + std::to_string(device) + " does not exist");
    }
    kw::DeviceGuard g(device);
    auto* q = new (std::nothrow) Queue;
    if (!q)
        return kw::resource("Queue: out of memory");
    q->device = device;
    q->flavor = flavor;
    cudaError_t e = cudaStreamCreateWithFlags(&q->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess)
        e = cudaStreamCreateWithFlags(&q->aux, cudaStreamNonBlocking);
    if (e == cudaSuccess)
        e = cudaStreamCreateWithFlags(&q->h2d, cudaStreamNonBlocking);
    if (e == cudaSuccess)
        e = cudaStreamCreateWithFlags(&q->comp2, cudaStreamNonBlocking);
    for (int i = 0; e == cudaSuccess && i < Queue::kRing; ++i) {
        e = cudaEventCreateWithFlags(&q->ev_ready[i], cudaEventDisableTiming);
        if (e == cudaSuccess)
            e = cudaEventCreateWithFlags(&q->ev_free[i], cudaEventDisableTiming);
        if (e == cudaSuccess)
            e = cudaEventCreateWithFlags(&q->ev_h2d[i], cudaEventDisableTiming);
    }
    if (e == cudaSuccess)
        e = cudaEventCreateWithFlags(&q->ev_join, cudaEventDisableTiming);
    if (e == cudaSuccess)
        e = cudaEventCreateWithFlags(&q->ev_join2, cudaEventDisableTiming);
    if (e == cudaSuccess)
        e = cudaEventCreateWithFlags(&q->ev_start, cudaEventDisableTiming);
    if (e == cudaSuccess)
        e = cudaEventCreateWithFlags(&q->ev_b, cudaEventDisableTiming);
    for (int i = 0; e == cudaSuccess && i < Queue::kBPanels; ++i)
        e = cudaEventCreateWithFlags(&q->ev_bp[i], cudaEventDisableTiming);
    if (e != cudaSuccess) {
        cudaGetLastError();
        delete q;
        return kw::resource(std::string("Queue: stream creation failed: ") + cudaGetErrorString(e));
    }
    *out = reinterpret_cast<kw_queue>(q);
    return KW_OK;
}

kw_status kw_queue_destroy(kw_queue qh)
{
    if (!qh)
        return KW_OK;
    auto* q = reinterpret_cast<Queue*>(qh);
    kw::DeviceGuard g(q->device);
    cudaStreamSynchronize(q->stream);
    cudaStreamSynchronize(q->aux);
    cudaStreamSynchronize(q->h2d);
    for (int i = 0; i < Queue::kRing; ++i) {
        if (q->ev_ready[i])
            cudaEventDestroy(q->ev_ready[i]);
        if (q->ev_free[i])
            cudaEventDestroy(q->ev_free[i]);
        if (q->ev_h2d[i])
            cudaEventDestroy(q->ev_h2d[i]);
    }
    for (cudaEvent_t e : {q->ev_join, q->ev_join2, q->ev_start, q->ev_b})
        if (e)
            cudaEventDestroy(e);
    for (cudaEvent_t e : q->ev_bp)
        if (e)
            cudaEventDestroy(e);
    {
        auto slots = kw::take_slots(q);
        if (q->staged)
            kw::release_slot(*q->staged);
        kw::resolve_slots(q, slots, false);
    }
    if (q->ev_order)
        cudaEventDestroy(q->ev_order);
    if (q->order_host)
        cudaFreeHost(q->order_host);
    if (q->order_dev)
        cudaFree(q->order_dev);
    if (q->scratch)
        cudaFree(q->scratch);
    cudaStreamSynchronize(q->comp2);
    kw::split_release(q->stream);
    kw::split_release(q->comp2);
    cudaStreamDestroy(q->comp2);
    cudaStreamDestroy(q->h2d);
    cudaStreamDestroy(q->aux);
    cudaStreamDestroy(q->stream);
    delete q;
    return KW_OK;
}

kw_status kw_queue_wait(kw_queue qh)
{
    KW_NVTX("kw queue wait");
    if (!qh)
        return kw::usage("null queue");
    auto* q = reinterpret_cast<Queue*>(qh);
    kw::DeviceGuard g(q->device);
    auto slots = kw::take_slots(q); // armed before this drain starts: complete once it returns
    cudaError_t e = cudaStreamSynchronize(q->stream);
    if (e != cudaSuccess) {
        kw::resolve_slots(q, slots, false);
        kw::task_fail(q, std::string("stream: ") + cudaGetErrorString(e));
    }
    else
        kw::resolve_slots(q, slots, true);
    for (cudaStream_t st : {q->stream, q->comp2})
        if (kw::split_take_abort(st))
            kw::task_fail(q, "dgemm (split): a tail piece's head never parked (bounded wait timed out)");
    std::lock_guard<std::mutex> lock(q->mu);
    if (q->failed == 0)
        return KW_OK;
    // TaskError message format (error.hpp:30-33).
    std::string msg = q->failed == 1 ? "task failed: " + q->first_failure
                                     : std::to_string(q->failed) + " tasks failed; first: " + q->first_failure;
    q->failed = 0;
    q->first_failure.clear();
    kw::set_error(msg);
    return KW_TASK;
}

kw_status kw_queue_report(kw_queue qh)
{
    if (!qh)
        return kw::usage("null queue");
    auto* q = reinterpret_cast<Queue*>(qh);
    if (q->flavor != KW_QUEUE_SYNC)
        return kw::usage("kw_queue_report: only a Sync queue's tasks are complete when their call returns");
    {
        std::lock_guard<std::mutex> lock(q->mu);
        if (q->failed == 0)
            return KW_OK;
    }
    // a failed task may have left work behind it: drain before reporting, as kw_queue_wait does
    return kw_queue_wait(qh);
}

kw_status kw_queue_device(kw_queue qh, int* device)
{
    if (!qh || !device)
        return kw::usage("kw_queue_device: null argument");
    *device = reinterpret_cast<Queue*>(qh)->device;
    return KW_OK;
}

kw_status kw_queue_flavor(kw_queue qh, int* flavor)
{
    if (!qh || !flavor)
        return kw::usage("kw_queue_flavor: null argument");
    *flavor = reinterpret_cast<Queue*>(qh)->flavor;
    return KW_OK;
}

kw_status kw_queue_stream(kw_queue qh, void** stream)
{
    if (!qh || !stream)
        return kw::usage("kw_queue_stream: null argument");
    *stream = reinterpret_cast<Queue*>(qh)->stream;
    return KW_OK;
}

kw_status kw_queue_shutdown(kw_queue qh)
{
    if (!qh)
        return kw::usage("null queue");
    auto* q = reinterpret_cast<Queue*>(qh);
    kw::DeviceGuard g(q->device);
    cudaStreamSynchronize(q->stream);
    q->shut = true;
    return KW_OK;
}

namespace {
// Arms (or, after a failed launch, drops) the slot staged for the launch that just happened and
// completes the enqueue like every other entry point.
kw_status finish_launch(Queue* q, std::shared_ptr<kw::FailSlot> slot, int cuda_error, const char* what)
{
    const std::string w = what ? what : "kernel";
    if (cuda_error != 0) {
        if (slot)
            kw::release_slot(*slot);
        cudaGetLastError();
        return kw::task_fail(q, w + ": " + cudaGetErrorString(static_cast<cudaError_t>(cuda_error)));
    }
    if (slot)
        kw::arm_slot(q, std::move(slot));
    kw::g_launches.fetch_add(1, std::memory_order_relaxed);
    kw::DeviceGuard g(q->device);
    return kw::after_enqueue(q, w.c_str());
}

// Slot of the legacy kw_queue_fail_slot / kw_queue_complete_launch pair, per calling thread.
thread_local Queue* t_legacy_queue = nullptr;
thread_local std::shared_ptr<kw::FailSlot> t_legacy_slot;
} // namespace

kw_status kw_queue_begin_launch(kw_queue qh, const char* what, void** stream, int* device, uint32_t** slot)
{
    if (!qh || !stream || !device || !slot)
        return kw::usage("kw_queue_begin_launch: null argument");
    auto* q = reinterpret_cast<Queue*>(qh);
    q->enqueue.lock(); // held until kw_queue_end_launch: the launch is one FIFO enqueue
    if (q->shut) {
        q->enqueue.unlock();
        return kw::usage("queue: enqueue after shutdown");
    }
    auto fs = kw::make_slot(what ? what : "kernel");
    if (!fs) {
        q->enqueue.unlock();
        return kw::resource("kw_queue_begin_launch: mapped pinned allocation failed");
    }
    q->staged = fs;
    *stream = q->stream;
    *device = q->device;
    *slot = fs->slot; // mapped + UVA: the host address is the device address
    return KW_OK;
}

kw_status kw_queue_end_launch(kw_queue qh, int cuda_error, const char* what)
{
    if (!qh)
        return kw::usage("null queue");
    auto* q = reinterpret_cast<Queue*>(qh);
    std::lock_guard<std::mutex> held(q->enqueue, std::adopt_lock);
    auto fs = std::move(q->staged);
    q->staged.reset();
    return finish_launch(q, std::move(fs), cuda_error, what);
}

kw_status kw_queue_complete_launch(kw_queue qh, int cuda_error, const char* what)
{
    if (!qh)
        return kw::usage("null queue");
    auto* q = reinterpret_cast<Queue*>(qh);
    std::shared_ptr<kw::FailSlot> fs;
    if (t_legacy_queue == q) {
        fs = std::move(t_legacy_slot);
        t_legacy_slot.reset();
        t_legacy_queue = nullptr;
    }
    return finish_launch(q, std::move(fs), cuda_error, what);
}

kw_status kw_queue_fail_slot(kw_queue qh, const char* what, uint32_t** slot)
{
    if (!qh || !slot)
        return kw::usage("kw_queue_fail_slot: null argument");
    auto* q = reinterpret_cast<Queue*>(qh);
    if (q->shut)
        return kw::usage("queue: enqueue after shutdown");
    auto fs = kw::make_slot(what ? what : "kernel");
    if (!fs)
        return kw::resource("kw_queue_fail_slot: mapped pinned allocation failed");
    if (t_legacy_slot)
        kw::release_slot(*t_legacy_slot); // staged but never launched
    t_legacy_queue = q;
    t_legacy_slot = fs;
    *slot = fs->slot;
    return KW_OK;
}

// ---- task events --------------------------------------------------------------------------

namespace {
kw_status record_event(kw_queue qh, kw_event* out, bool timing)
{
    KW_CHECK_QUEUE(qh);
    KW_ENQUEUE_LOCK(qh);
    if (!out)
        return kw::usage(timing ? "kw_event_record: null output" : "kw_task_marker: null output");
    auto* q = reinterpret_cast<Queue*>(qh);
    kw::DeviceGuard g(q->device);
    auto* ev = new kw_event_s{q->device, nullptr, q, nullptr, timing};
    {
        std::lock_guard<std::mutex> lock(q->mu);
        ev->slot = std::move(q->last_slot);
        q->last_slot.reset();
    }
    cudaError_t e = timing ? cudaEventCreate(&ev->ev) : cudaEventCreateWithFlags(&ev->ev, cudaEventDisableTiming);
    if (e == cudaSuccess)
        e = cudaEventRecord(ev->ev, q->stream);
    if (e != cudaSuccess) {
        if (ev->ev)
            cudaEventDestroy(ev->ev);
        delete ev;
        return kw::cuda_fail("event record", e);
    }
    *out = ev;
    return KW_OK;
}
} // namespace

kw_status kw_event_record(kw_queue qh, kw_event* out) { return record_event(qh, out, true); }

kw_status kw_task_marker(kw_queue qh, kw_event* out) { return record_event(qh, out, false); }

kw_status kw_event_state(kw_event ev, int* state)
{
    if (!ev || !state)
        return kw::usage("kw_event_state: null argument");
    kw::DeviceGuard g(ev->device);
    cudaError_t e = cudaEventQuery(ev->ev);
    if (e == cudaErrorNotReady) {
        cudaGetLastError();
        *state = KW_TASK_PENDING;
        return KW_OK;
    }
    // A task's own launch failure is returned synchronously by its kw_* call (and collected for
    // kw_queue_wait); the event reports completion, a device-side failure its functor recorded
    // (kw_queue_fail_slot), or a device fault (sticky, context-wide).
    if (e != cudaSuccess) {
        *state = KW_TASK_FAILED;
        return KW_OK;
    }
    *state = ev->slot && ev->slot->read() != 0 ? KW_TASK_FAILED : KW_TASK_DONE;
    return KW_OK;
}

kw_status kw_event_destroy(kw_event ev)
{
    if (!ev)
        return KW_OK;
    kw::DeviceGuard g(ev->device);
    cudaEventDestroy(ev->ev);
    delete ev;
    return KW_OK;
}

kw_status kw_event_elapsed_ms(kw_event a, kw_event b, float* ms)
{
    if (!a || !b || !ms)
        return kw::usage("kw_event_elapsed_ms: null argument");
    if (!a->timing || !b->timing)
        return kw::usage("kw_event_elapsed_ms: task markers carry no timestamp (use kw_event_record)");
    kw::DeviceGuard g(a->device);
    cudaError_t e = cudaEventSynchronize(b->ev);
    if (e == cudaSuccess)
        e = cudaEventElapsedTime(ms, a->ev, b->ev);
    return e == cudaSuccess ? KW_OK : kw::cuda_fail("event elapsed", e);
}

// ---- copies -------------------------------------------------------------------------------

kw_status kw_copy(kw_queue qh, void* dst, size_t dst_pitch, const size_t dst_extent[3], const void* src,
                  size_t src_pitch, const size_t src_extent[3], uint32_t dim, const size_t extent[3],
                  size_t elem_size)
{
    KW_CHECK_QUEUE(qh);
    KW_ENQUEUE_LOCK(qh);
    KW_NVTX("kw copy");
    auto* q = reinterpret_cast<Queue*>(qh);
    if (dim < 1 || dim > 3)
        return kw::usage("copy: buffer and extent dimensionalities must match");
    if (!dst || !src || !extent || !dst_extent || !src_extent)
        return kw::usage("copy: null argument");
    if (elem_size == 0)
        return kw::usage("copy: element sizes must match");
    for (uint32_t k = 0; k < dim; ++k)
        if (extent[k] > dst_extent[k] || extent[k] > src_extent[k])
            return kw::usage("copy: extent exceeds a buffer extent");
    size_t line = 0, dst_row = 0, src_row = 0;
    if (__builtin_mul_overflow(extent[dim - 1], elem_size, &line) ||
        __builtin_mul_overflow(dst_extent[dim - 1], elem_size, &dst_row) ||
        __builtin_mul_overflow(src_extent[dim - 1], elem_size, &src_row))
        return kw::usage("copy: row size overflows the address space");
    if (dim > 1 && (dst_pitch < dst_row || src_pitch < src_row))
        return kw::usage("copy: row pitch smaller than a row");
    for (uint32_t k = 0; k < dim; ++k)
        if (extent[k] == 0)
            return KW_OK;
    kw::DeviceGuard g(q->device);
    cudaError_t e = cudaSuccess;
    if (dim == 1) {
        e = cudaMemcpyAsync(dst, src, line, cudaMemcpyDefault, q->stream);
    }
    else if (dim == 2) {
        e = cudaMemcpy2DAsync(dst, dst_pitch, src, src_pitch, line, extent[0], cudaMemcpyDefault, q->stream);
    }
    else {
        // 3-D: each side's row index is (i0 * ext[1] + i1) with its OWN extent (buffer.cpp:124-139),
        // i.e. a pitched volume whose slice height is that side's extent[1].
        cudaMemcpy3DParms p = {};
        p.srcPtr = make_cudaPitchedPtr(const_cast<void*>(src), src_pitch, src_extent[2] * elem_size, src_extent[1]);
        p.dstPtr = make_cudaPitchedPtr(dst, dst_pitch, dst_extent[2] * elem_size, dst_extent[1]);
        p.extent = make_cudaExtent(line, extent[1], extent[0]);
        p.kind = cudaMemcpyDefault;
        e = cudaMemcpy3DAsync(&p, q->stream);
    }
    if (e != cudaSuccess)
        return kw::task_fail(q, std::string("copy: ") + cudaGetErrorString(e));
    return kw::after_enqueue(q, "copy");
}

// ---- work division ------------------------------------------------------------------------

kw_status kw_total_extent(const kw_workdiv* wd, int origin, int unit, size_t out[3])
{
    if (!wd || !out)
        return kw::usage("totalExtent: null argument");
    if (wd->dim < 1 || wd->dim > 3)
        return kw::usage("IndexVec: dimensionality must be 1, 2 or 3");
    for (int k = 0; k < 3; ++k)
        out[k] = 1;
    for (uint32_t k = 0; k < wd->dim; ++k) {
        size_t v;
        if (origin == 0 && unit == 0)
            v = wd->blocks[k];
        else if (origin == 0 && unit == 1)
            v = wd->blocks[k] * wd->threads[k];
        else if (origin == 0 && unit == 2)
            v = wd->blocks[k] * wd->threads[k] * wd->elems[k];
        else if (origin == 1 && unit == 1)
            v = wd->threads[k];
        else if (origin == 1 && unit == 2)
            v = wd->threads[k] * wd->elems[k];
        else if (origin == 2 && unit == 2)
            v = wd->elems[k];
        else
            return kw::usage("totalExtent: unsupported (origin, unit) pair");
        out[k] = v;
    }
    return KW_OK;
}

kw_status kw_divide_for_gpu(uint32_t dim, const size_t problem[3], const size_t threads_hint[3],
                            const size_t elems_hint[3], kw_workdiv* out)
{
    if (!problem || !threads_hint || !elems_hint || !out)
        return kw::usage("divideForBackend: null argument");
    if (dim < 1 || dim > 3)
        return kw::usage("IndexVec: dimensionality must be 1, 2 or 3");
    kw_workdiv wd = {};
    wd.dim = dim;
    for (int k = 0; k < 3; ++k)
        wd.blocks[k] = wd.threads[k] = wd.elems[k] = 1;
    for (uint32_t k = 0; k < dim; ++k) {
        if (problem[k] == 0)
            return kw::usage("WorkDiv: problem extent has a zero component; every level extent is at least 1");
        if (threads_hint[k] == 0)
            return kw::usage("WorkDiv: threadsPerBlock hint has a zero component; every level extent is at least 1");
        if (elems_hint[k] == 0)
            return kw::usage("WorkDiv: elementsPerThread hint has a zero component; every level extent is at least 1");
        wd.threads[k] = threads_hint[k];
        wd.elems[k] = elems_hint[k];
        wd.blocks[k] = kw::ceil_div(problem[k], threads_hint[k] * elems_hint[k]);
    }
    *out = wd;
    return KW_OK;
}

uint64_t kw_launch_count(void) { return kw::g_launches.load(); }

kw_status kw_l2_flush(kw_queue qh)
{
    KW_CHECK_QUEUE(qh);
    KW_ENQUEUE_LOCK(qh);
    auto* q = reinterpret_cast<Queue*>(qh);
    static void* flush_buf[64] = {}; // per device: 2 x L2 bytes, written once per call
    static size_t flush_bytes[64] = {};
    static std::mutex mu;
    if (q->device >= 64)
        return kw::usage("l2 flush: device index beyond 63");
    kw::DeviceGuard g(q->device);
    std::lock_guard<std::mutex> lock(mu);
    if (!flush_buf[q->device]) {
        int l2 = 0;
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, q->device);
        size_t bytes = static_cast<size_t>(l2) * 2;
        if (cudaMalloc(&flush_buf[q->device], bytes) != cudaSuccess) {
            cudaGetLastError();
            return kw::resource("L2 flush buffer allocation failed");
        }
        flush_bytes[q->device] = bytes;
    }
    cudaError_t e = cudaMemsetAsync(flush_buf[q->device], 0, flush_bytes[q->device], q->stream);
    if (e != cudaSuccess)
        return kw::task_fail(q, std::string("l2 flush: ") + cudaGetErrorString(e));
    return kw::after_enqueue(q, "l2 flush");
}

} // extern "C"
