"""B200-native (sm_100a) kernelweave hot path: AXPY and tiled DGEMM behind the reference's
kernel-functor API. The compute lives in libkw_b200.so (hand-written CUDA, C-ABI in
include/kw_b200.h); this package is the Python mirror of the reference interface used by the
tests, the bench and smoke()."""
from . import _lib  # noqa: F401
from .kernelweave import (  # noqa: F401
    AxpyArgs, AxpyKernel, BackendKind, Buffer, CopyTask, Device, ExecTask, GemmArgs, GemmNaiveKernel,
    GemmTiledKernel, IndexVec, Level, Queue, QueueFlavor, ResourceError, TaskError, TaskHandle, TaskState,
    Unit, UsageError, WorkDiv, allocBuffer, axpyWorkDiv, copyBuffer, createCopy, createExec, divideForBackend,
    executeTask, gemmNaiveWorkDiv, gemmTiledWorkDiv, totalExtent,
)

__all__ = [n for n in dir() if not n.startswith("_")]
