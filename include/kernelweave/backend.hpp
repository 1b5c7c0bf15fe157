/* kernelweave B200 drop-in — back-end kinds (reference: core/include/kernelweave/backend.hpp).
 * GpuCudaRt (the paper's AccGpuCudaRt) is the only kind that executes in this
 * build; the CPU kinds are kept for source compatibility of divideForBackend (pure host
 * arithmetic). Executing on them throws UsageError: there is no CPU fallback. */
#pragma once

#include "kernelweave/error.hpp"

#include <array>
#include <string_view>

namespace kernelweave {

enum class BackendKind {
    Serial,
    BlocksParallel,
    ThreadsParallel,
    GpuCudaRt,
};

/// The back-ends that execute tasks in this build.
inline constexpr std::array<BackendKind, 1> allBackends{BackendKind::GpuCudaRt};

inline std::string_view backendName(BackendKind kind)
{
    switch (kind) {
    case BackendKind::Serial:
        return "serial";
    case BackendKind::BlocksParallel:
        return "blocks";
    case BackendKind::ThreadsParallel:
        return "threads";
    case BackendKind::GpuCudaRt:
        return "gpu";
    }
    return "?";
}

inline BackendKind parseBackend(std::string_view name)
{
    for (BackendKind k : {BackendKind::Serial, BackendKind::BlocksParallel, BackendKind::ThreadsParallel,
                          BackendKind::GpuCudaRt})
        if (backendName(k) == name)
            return k;
    throw UsageError("unknown backend '" + std::string(name) + "'");
}

namespace detail {
inline void requireGpu(BackendKind kind)
{
    if (kind != BackendKind::GpuCudaRt)
        throw UsageError("back-end '" + std::string(backendName(kind)) +
                         "' does not exist in the B200 build (no CPU fallback); use BackendKind::GpuCudaRt");
}
} // namespace detail

} // namespace kernelweave
