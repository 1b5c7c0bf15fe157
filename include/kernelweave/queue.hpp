/* kernelweave B200 drop-in — queues and tasks (reference: core/include/kernelweave/queue.hpp).
 * A Queue is a CUDA stream on one GPU (kw_queue). Sync: every enqueue completes before it
 * returns; Async: enqueue returns immediately. Usage errors are thrown before anything is
 * enqueued; failed tasks are collected and reported by wait() as TaskError (queue.hpp:86-137). */
#pragma once

#include "kernelweave/device.hpp"
#include "kernelweave/work_div.hpp"

#include <exception>
#include <functional>
#include <memory>
#include <mutex>
#include <tuple>
#include <type_traits>
#include <utility>

namespace kernelweave {

enum class QueueFlavor { Sync, Async };
enum class TaskState { Pending, Running, Done, Failed };

/// Non-blocking view of one enqueued task (queue.hpp:36-52): a CUDA event recorded after it.
class TaskHandle {
public:
    TaskState state() const
    {
        if (!m_event) // a Sync queue's task: complete when enqueue returned
            return m_failed || !m_completed ? TaskState::Failed : TaskState::Done;
        int s = 0;
        detail::check(kw_event_state(m_event.get(), &s));
        if (m_failed)
            return TaskState::Failed;
        return static_cast<TaskState>(s);
    }
    std::exception_ptr error() const
    {
        return state() == TaskState::Failed
                   ? std::make_exception_ptr(TaskError(1, m_message.empty() ? "task failed on the device" : m_message))
                   : nullptr;
    }

private:
    friend class Queue;
    TaskHandle(kw_event ev, bool failed, std::string msg, bool completed = false)
        : m_event(ev, [](kw_event e) {
              if (e)
                  kw_event_destroy(e);
          }),
          m_failed(failed), m_completed(completed), m_message(std::move(msg))
    {
    }
    std::shared_ptr<kw_event_s> m_event;
    bool m_failed;
    bool m_completed;
    std::string m_message;
};

/// Binding of back-end, division, kernel and arguments (queue.hpp:63-67). The body enqueues the
/// kernel on a kw_queue; constructing a task executes nothing.
struct ExecTask {
    BackendKind backend;
    WorkDiv workDiv;
    std::function<kw_status(kw_queue)> body;
};

/// An enqueueable deep copy built by createCopy().
struct CopyTask {
    std::function<kw_status(kw_queue)> body;
};

namespace detail {
/// Maps a kernel functor type onto its sm_100a launch. Specialised by the shipped kernels
/// (kernels/axpy.hpp, kernels/gemm.hpp → libkw_b200.so entry points) and, for user functors
/// compiled by nvcc, by KW_DEVICE_FUNCTOR (kernelweave/cuda_exec.cuh). Contract:
///   static void validate(const WorkDiv&, const Args&...);          // throws UsageError
///   static kw_status launch(kw_queue, const WorkDiv&, const Kernel&, const Args&...);
///   static Device device(const Args&...);                            // for executeTask
template <class Kernel, class... Args>
struct Launcher {
    static_assert(sizeof(Kernel) == 0,
                  "no sm_100a launcher is registered for this kernel functor: compile the translation unit "
                  "with nvcc, include kernelweave/cuda_exec.cuh and declare KW_DEVICE_FUNCTOR(YourKernel)");
};
} // namespace detail

/// queue.hpp:74-82. Arguments are validated now (UsageError before anything is enqueued) and
/// stored by value; the buffers they point to must outlive the task.
template <class Kernel, class... Args>
ExecTask createExec(BackendKind backend, const WorkDiv& wd, Kernel kernel, Args... args)
{
    detail::requireGpu(backend);
    detail::Launcher<Kernel, Args...>::validate(wd, args...);
    return ExecTask{backend, wd, [wd, kernel, bound = std::make_tuple(std::move(args)...)](kw_queue q) {
                        return std::apply(
                            [&](const auto&... a) {
                                return detail::Launcher<Kernel, Args...>::launch(q, wd, kernel, a...);
                            },
                            bound);
                    }};
}

class Queue {
public:
    Queue(Device device, QueueFlavor flavor) : m_device(device), m_flavor(flavor)
    {
        const int cuda = device.isHost() ? 0 : device.cudaIndex(); // host copies use GPU 0's engines
        kw_queue q = nullptr;
        detail::check(kw_queue_create(cuda, flavor == QueueFlavor::Sync ? KW_QUEUE_SYNC : KW_QUEUE_ASYNC, &q));
        m_q = q;
    }
    ~Queue()
    {
        if (m_q)
            kw_queue_destroy(m_q);
    }
    Queue(const Queue&) = delete;
    Queue& operator=(const Queue&) = delete;

    TaskHandle enqueue(ExecTask task) { return run(task.body); }
    TaskHandle enqueue(CopyTask task) { return run(task.body); }

    /// Blocks until everything enqueued so far completed; throws TaskError for failures since
    /// the last report (queue.cpp:99-131). Idempotent.
    void wait() { detail::check(kw_queue_wait(m_q)); }
    /// Sync queues: throws the TaskError of failed tasks since the last report without a stream
    /// round trip (their tasks completed inside enqueue).
    void report() { detail::check(kw_queue_report(m_q)); }
    void shutdown() { detail::check(kw_queue_shutdown(m_q)); }

    Device device() const noexcept { return m_device; }
    QueueFlavor flavor() const noexcept { return m_flavor; }
    kw_queue native() const noexcept { return m_q; }

private:
    TaskHandle run(const std::function<kw_status(kw_queue)>& body)
    {
        std::lock_guard<std::mutex> lock(m_mu); // arrival order at the lock is the FIFO order
        const kw_status st = body(m_q);
        if (st == KW_USAGE || st == KW_RESOURCE)
            detail::check(st);
        const std::string msg = st == KW_TASK ? kw_last_error() : "";
        // A Sync queue completed the task inside the call (queue.cpp:21-23): its handle needs no
        // event — recording one would add a GPU round trip to the next wait().
        if (m_flavor == QueueFlavor::Sync)
            return TaskHandle(nullptr, st == KW_TASK, msg, true);
        kw_event ev = nullptr;
        if (kw_task_marker(m_q, &ev) != KW_OK)
            ev = nullptr;
        return TaskHandle(ev, st == KW_TASK, msg);
    }

    Device m_device;
    QueueFlavor m_flavor;
    kw_queue m_q = nullptr;
    std::mutex m_mu;
};

} // namespace kernelweave
