/* kernelweave B200 drop-in — executeTask (reference: core/include/kernelweave/exec.hpp:32-36).
 * Externally synchronous: the task runs on a per-device Sync queue and completes (or throws)
 * before the call returns. The reference's detail::runGrid seam is replaced by the sm_100a
 * launchers of libkw_b200.so (detail::Launcher). */
#pragma once

#include "kernelweave/queue.hpp"

#include <map>
#include <memory>
#include <mutex>

namespace kernelweave {

namespace detail {
inline Queue& defaultQueue(Device device)
{
    static std::mutex mu;
    static std::map<int, std::unique_ptr<Queue>> queues;
    std::lock_guard<std::mutex> lock(mu);
    auto& q = queues[device.index()];
    if (!q)
        q = std::make_unique<Queue>(device, QueueFlavor::Sync);
    return *q;
}
} // namespace detail

template <class Kernel, class... Args>
void executeTask(BackendKind backend, const WorkDiv& wd, const Kernel& kernel, const Args&... args)
{
    ExecTask task = createExec(backend, wd, kernel, args...);
    Queue& q = detail::defaultQueue(detail::Launcher<Kernel, Args...>::device(args...));
    q.enqueue(std::move(task));
    q.report(); // the Sync queue already completed the task: no second stream round trip
}

} // namespace kernelweave
