"""Python mirror of the kernelweave kernel-functor API over the B200 C-ABI.

Same names, argument meaning and error behaviour as the reference (paths relative to
/root/reference/proj/core/include/kernelweave):
  IndexVec (index_vec.hpp:25-97), Level / Unit / WorkDiv / totalExtent / divideForBackend
  (work_div.hpp:13-75), BackendKind (backend.hpp:23-40), Device (device.hpp:14-37), Buffer /
  allocBuffer / createCopy / copyBuffer (buffer.hpp:29-144), Queue / QueueFlavor / TaskState /
  TaskHandle / ExecTask / CopyTask / createExec (queue.hpp:21-137), executeTask (exec.hpp:32-36),
  AxpyKernel / AxpyArgs / axpyWorkDiv (kernels/axpy.hpp), GemmTiledKernel / GemmNaiveKernel /
  GemmArgs / gemmTiledWorkDiv / gemmNaiveWorkDiv (kernels/gemm.hpp), and the error taxonomy
  UsageError / ResourceError / TaskError (error.hpp).

B200 back-end: `BackendKind.GpuCudaRt` (the paper's AccGpuCudaRt accelerator)
is the only kind that executes in this build. The CPU kinds are kept so the reference's
`divideForBackend` arithmetic (pure host code) stays source compatible; executing a task on
them raises UsageError — there is no CPU fallback. `Device.host()` buffers are page-locked host
memory; executing a kernel on them streams the data through the GPU (the e2e path).
"""
from __future__ import annotations

import ctypes as C
import enum
import threading
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from . import _lib as L


# ---- errors (error.hpp) ------------------------------------------------------------------
class UsageError(ValueError):
    """A caller violated an API precondition (error.hpp:13)."""


class ResourceError(RuntimeError):
    """A system resource could not be obtained (error.hpp:19)."""


class TaskError(RuntimeError):
    """Raised by Queue.wait() when tasks failed since the last report (error.hpp:26-40)."""

    def __init__(self, failed_count: int, message: str):
        super().__init__(message)
        self._failed = failed_count

    def failedCount(self) -> int:
        return self._failed


def _raise_for(status: int) -> None:
    if status == L.KW_OK:
        return
    msg = L.last_error()
    if status == L.KW_USAGE:
        raise UsageError(msg)
    if status == L.KW_RESOURCE:
        raise ResourceError(msg)
    n = 1
    if " tasks failed" in msg:
        try:
            n = int(msg.split(" ", 1)[0])
        except ValueError:
            n = 1
    raise TaskError(n, msg)


# ---- IndexVec (index_vec.hpp) ---------------------------------------------------------------
class IndexVec:
    """1-3 non-negative components, slowest first; the last component varies fastest."""

    maxDim = 3
    __slots__ = ("_c",)

    def __init__(self, *comps: int):
        if len(comps) == 1 and isinstance(comps[0], (tuple, list)):
            comps = tuple(comps[0])
        if not 1 <= len(comps) <= 3:
            raise UsageError("IndexVec: dimensionality must be 1, 2 or 3")
        for v in comps:
            if int(v) < 0:
                raise UsageError("IndexVec: components are non-negative")
        self._c = tuple(int(v) for v in comps)

    @staticmethod
    def filled(dim: int, value: int) -> "IndexVec":
        if not 1 <= dim <= 3:
            raise UsageError("IndexVec: dimensionality must be 1, 2 or 3")
        return IndexVec(*([value] * dim))

    def dim(self) -> int:
        return len(self._c)

    def __getitem__(self, k: int) -> int:
        if not isinstance(k, int) or k < 0 or k >= len(self._c):
            raise UsageError("IndexVec: component index out of range")
        return self._c[k]

    def product(self) -> int:
        p = 1
        for v in self._c:
            p *= v
        return p

    def with_(self, k: int, value: int) -> "IndexVec":
        if k < 0 or k >= len(self._c):
            raise UsageError("IndexVec: component index out of range")
        c = list(self._c)
        c[k] = value
        return IndexVec(*c)

    def tuple(self) -> tuple:
        return self._c

    def __eq__(self, other) -> bool:
        return isinstance(other, IndexVec) and self._c == other._c

    def __hash__(self) -> int:
        return hash(self._c)

    def __mul__(self, other: "IndexVec") -> "IndexVec":
        return elementwiseProduct(self, other)

    def __add__(self, other: "IndexVec") -> "IndexVec":
        return elementwiseSum(self, other)

    def __repr__(self) -> str:
        return "(" + ", ".join(map(str, self._c)) + ")"


def _same_dim(a: IndexVec, b: IndexVec, what: str) -> None:
    if a.dim() != b.dim():
        raise UsageError(f"{what}: dimensionality mismatch ({a.dim()} vs {b.dim()})")


def elementwiseProduct(a: IndexVec, b: IndexVec) -> IndexVec:
    _same_dim(a, b, "elementwiseProduct")
    return IndexVec(*(x * y for x, y in zip(a.tuple(), b.tuple())))


def elementwiseSum(a: IndexVec, b: IndexVec) -> IndexVec:
    _same_dim(a, b, "elementwiseSum")
    return IndexVec(*(x + y for x, y in zip(a.tuple(), b.tuple())))


def ceilDivide(a: IndexVec, b: IndexVec) -> IndexVec:
    _same_dim(a, b, "ceilDivide")
    if any(y == 0 for y in b.tuple()):
        raise UsageError("ceilDivide: zero divisor component")
    return IndexVec(*((x + y - 1) // y for x, y in zip(a.tuple(), b.tuple())))


def insideExtent(idx: IndexVec, extent: IndexVec) -> bool:
    _same_dim(idx, extent, "insideExtent")
    return all(i < e for i, e in zip(idx.tuple(), extent.tuple()))


def linearize(idx: IndexVec, extent: IndexVec) -> int:
    _same_dim(idx, extent, "linearize")
    lin = 0
    for i, e in zip(idx.tuple(), extent.tuple()):
        if i >= e:
            raise UsageError("linearize: index component out of range")
        lin = lin * e + i
    return lin


def delinearize(lin: int, extent: IndexVec) -> IndexVec:
    if lin >= extent.product():
        raise UsageError("delinearize: linear index out of range")
    comps = []
    for e in reversed(extent.tuple()[1:]):
        comps.append(lin % e)
        lin //= e
    comps.append(lin)
    return IndexVec(*reversed(comps))


# ---- work division (work_div.hpp / work_div.cpp) ------------------------------------------
class Level(enum.Enum):
    Grid = 0
    Block = 1
    Thread = 2


class Unit(enum.Enum):
    Blocks = 0
    Threads = 1
    Elems = 2


class BackendKind(enum.Enum):
    Serial = 0
    BlocksParallel = 1
    ThreadsParallel = 2
    GpuCudaRt = 3  # the B200 accelerator (this build's only executable kind)


allBackends = (BackendKind.GpuCudaRt,)


def backendName(kind: BackendKind) -> str:
    return {BackendKind.Serial: "serial", BackendKind.BlocksParallel: "blocks",
            BackendKind.ThreadsParallel: "threads", BackendKind.GpuCudaRt: "gpu"}[kind]


def parseBackend(name: str) -> BackendKind:
    for k in BackendKind:
        if backendName(k) == name:
            return k
    raise UsageError(f"unknown backend '{name}'")


class WorkDiv:
    """WorkDiv{blocksPerGrid, threadsPerBlock, elementsPerThread} (work_div.hpp:33-53)."""

    def __init__(self, blocksPerGrid: IndexVec, threadsPerBlock: IndexVec, elementsPerThread: IndexVec):
        _same_dim(blocksPerGrid, threadsPerBlock, "WorkDiv")
        _same_dim(blocksPerGrid, elementsPerThread, "WorkDiv")
        for name, v in (("blocksPerGrid", blocksPerGrid), ("threadsPerBlock", threadsPerBlock),
                        ("elementsPerThread", elementsPerThread)):
            if any(c == 0 for c in v.tuple()):
                raise UsageError(f"WorkDiv: {name} has a zero component; every level extent is at least 1")
        self._b, self._t, self._e = blocksPerGrid, threadsPerBlock, elementsPerThread

    def blocksPerGrid(self) -> IndexVec:
        return self._b

    def threadsPerBlock(self) -> IndexVec:
        return self._t

    def elementsPerThread(self) -> IndexVec:
        return self._e

    def dim(self) -> int:
        return self._b.dim()

    def __eq__(self, o) -> bool:
        return isinstance(o, WorkDiv) and (self._b, self._t, self._e) == (o._b, o._t, o._e)

    def __repr__(self) -> str:
        return f"WorkDiv(blocks={self._b}, threads={self._t}, elems={self._e})"

    def to_c(self) -> L.kw_workdiv:
        wd = L.kw_workdiv()
        wd.dim = self.dim()
        wd.blocks = L.sz3(self._b.tuple())
        wd.threads = L.sz3(self._t.tuple())
        wd.elems = L.sz3(self._e.tuple())
        return wd

    @staticmethod
    def from_c(wd: L.kw_workdiv) -> "WorkDiv":
        d = wd.dim
        return WorkDiv(IndexVec(*wd.blocks[:d]), IndexVec(*wd.threads[:d]), IndexVec(*wd.elems[:d]))


def totalExtent(wd: WorkDiv, origin: Level, unit: Unit) -> IndexVec:
    """work_div.cpp:65-94."""
    b, t, e = wd.blocksPerGrid(), wd.threadsPerBlock(), wd.elementsPerThread()
    table = {
        (Level.Grid, Unit.Blocks): lambda: b,
        (Level.Grid, Unit.Threads): lambda: b * t,
        (Level.Grid, Unit.Elems): lambda: b * t * e,
        (Level.Block, Unit.Threads): lambda: t,
        (Level.Block, Unit.Elems): lambda: t * e,
        (Level.Thread, Unit.Elems): lambda: e,
    }
    f = table.get((origin, unit))
    if f is None:
        raise UsageError(f"totalExtent: unsupported (origin, unit) pair ({origin.name}, {unit.name})")
    return f()


def divideForBackend(problemExtent: IndexVec, backend: BackendKind, threadsPerBlockHint: IndexVec,
                     elementsPerThreadHint: IndexVec) -> WorkDiv:
    """work_div.cpp:96-119; GpuCudaRt takes the thread-level shape ceil(N/(B*V)) x B x V."""
    _same_dim(problemExtent, threadsPerBlockHint, "divideForBackend")
    _same_dim(problemExtent, elementsPerThreadHint, "divideForBackend")
    for name, v in (("problem extent", problemExtent), ("threadsPerBlock hint", threadsPerBlockHint),
                    ("elementsPerThread hint", elementsPerThreadHint)):
        if any(c == 0 for c in v.tuple()):
            raise UsageError(f"WorkDiv: {name} has a zero component; every level extent is at least 1")
    ones = IndexVec.filled(problemExtent.dim(), 1)
    if backend in (BackendKind.Serial, BackendKind.BlocksParallel):
        return WorkDiv(ceilDivide(problemExtent, elementsPerThreadHint), ones, elementsPerThreadHint)
    if backend in (BackendKind.ThreadsParallel, BackendKind.GpuCudaRt):
        return WorkDiv(ceilDivide(problemExtent, threadsPerBlockHint * elementsPerThreadHint),
                       threadsPerBlockHint, elementsPerThreadHint)
    raise UsageError("divideForBackend: unknown BackendKind value")


# ---- devices (device.hpp) ---------------------------------------------------------------------
class Device:
    """Device 0 is the host; Device.logical(i + 1) is CUDA device i (the attach point the
    reference documents for real devices, device.hpp:10-13)."""

    __slots__ = ("_index",)

    def __init__(self, index: int = 0):
        if index < 0:
            raise UsageError("Device: negative device index")
        self._index = index

    @staticmethod
    def host() -> "Device":
        return Device(0)

    @staticmethod
    def logical(index: int) -> "Device":
        return Device(index)

    @staticmethod
    def gpu(cuda_index: int) -> "Device":
        return Device(cuda_index + 1)

    def index(self) -> int:
        return self._index

    def isHost(self) -> bool:
        return self._index == 0

    def cuda_index(self) -> int:
        return self._index - 1

    def __eq__(self, o) -> bool:
        return isinstance(o, Device) and o._index == self._index

    def __repr__(self) -> str:
        return "Device.host()" if self.isHost() else f"Device.gpu({self._index - 1})"


def device_count() -> int:
    n = C.c_int(0)
    st = L.lib().kw_device_count(C.byref(n))
    return n.value if st == L.KW_OK else 0


# ---- buffers (buffer.hpp / buffer.cpp) --------------------------------------------------------
_NP = {4: np.float32, 8: np.float64}


class Buffer:
    """Pitched n-D region on a device (or page-locked host memory for Device.host())."""

    defaultRowAlignment = 64

    def __init__(self, device: Device, extent: IndexVec, elemSize: int, rowAlignment: int = 64):
        if not isinstance(extent, IndexVec):
            extent = IndexVec(*extent) if isinstance(extent, (tuple, list)) else IndexVec(extent)
        self._device = device
        self._extent = extent
        self._elem = int(elemSize)
        ptr = C.c_void_p()
        pitch = C.c_size_t()
        _raise_for(L.lib().kw_buffer_alloc(-1 if device.isHost() else device.cuda_index(), extent.dim(),
                                           L.sz3(extent.tuple()), self._elem, int(rowAlignment),
                                           C.byref(ptr), C.byref(pitch)))
        self._ptr = ptr.value
        self._pitch = pitch.value

    def __del__(self):
        p = getattr(self, "_ptr", None)
        if p:
            try:
                L.lib().kw_buffer_free(-1 if self._device.isHost() else self._device.cuda_index(), p)
            except Exception:
                pass
            self._ptr = None

    def free(self) -> None:
        self.__del__()

    def device(self) -> Device:
        return self._device

    def extent(self) -> IndexVec:
        return self._extent

    def dim(self) -> int:
        return self._extent.dim()

    def elemSize(self) -> int:
        return self._elem

    def rowPitch(self) -> int:
        return self._pitch

    def rowCount(self) -> int:
        r = 1
        for v in self._extent.tuple()[:-1]:
            r *= v
        return r

    def rowBytes(self) -> int:
        return self._extent[self.dim() - 1] * self._elem

    def storageBytes(self) -> int:
        return self.rowCount() * self._pitch

    def data(self) -> int:
        return self._ptr

    def leadingDim(self) -> int:
        if self._pitch % self._elem:
            raise UsageError("Buffer: row pitch not divisible by element size")
        return self._pitch // self._elem

    # -- host-side convenience (tests / bench) --
    def host_view(self) -> np.ndarray:
        """Zero-copy numpy view of a host buffer (rows x pitch-in-elements, dtype by elemSize)."""
        if not self._device.isHost():
            raise UsageError("host_view: device buffer")
        raw = (C.c_char * self.storageBytes()).from_address(self._ptr)
        a = np.frombuffer(raw, dtype=_NP[self._elem])
        if self.dim() == 1:
            return a
        return a.reshape(self.rowCount(), self._pitch // self._elem)

    def upload(self, arr: np.ndarray, queue: Optional["Queue"] = None) -> None:
        """Copies a dense host array of this buffer's logical extent into the buffer."""
        arr = np.ascontiguousarray(arr, dtype=_NP[self._elem])
        ext = self._extent.tuple()
        if arr.size != self._extent.product():
            raise UsageError("upload: size mismatch")
        q = queue or _default_queue(self._device)
        _raise_for(L.lib().kw_copy(q._h, self._ptr, self._pitch, L.sz3(ext), arr.ctypes.data,
                                   ext[-1] * self._elem, L.sz3(ext), self.dim(), L.sz3(ext), self._elem))
        q.wait()

    def download(self, queue: Optional["Queue"] = None) -> np.ndarray:
        """Returns the logical extent as a dense numpy array (shape = extent)."""
        ext = self._extent.tuple()
        out = np.empty(ext, dtype=_NP[self._elem])
        q = queue or _default_queue(self._device)
        _raise_for(L.lib().kw_copy(q._h, out.ctypes.data, ext[-1] * self._elem, L.sz3(ext), self._ptr,
                                   self._pitch, L.sz3(ext), self.dim(), L.sz3(ext), self._elem))
        q.wait()
        return out

    def download_raw(self, queue: Optional["Queue"] = None) -> bytes:
        """Every byte of the storage (padding included) — for canary checks."""
        out = np.empty(self.storageBytes(), dtype=np.uint8)
        q = queue or _default_queue(self._device)
        n = self.storageBytes()
        _raise_for(L.lib().kw_copy(q._h, out.ctypes.data, n, L.sz3((n,)), self._ptr, n, L.sz3((n,)), 1,
                                   L.sz3((n,)), 1))
        q.wait()
        return out.tobytes()

    def fill_raw(self, byte: int, queue: Optional["Queue"] = None) -> None:
        q = queue or _default_queue(self._device)
        _raise_for(L.lib().kw_memset(q._h, self._ptr, byte, self.storageBytes()))
        q.wait()


def allocBuffer(device: Device, extent: IndexVec, elemSize: int, rowAlignment: int = 64) -> Buffer:
    return Buffer(device, extent, elemSize, rowAlignment)


# ---- queues and tasks (queue.hpp) -------------------------------------------------------------
class QueueFlavor(enum.Enum):
    Sync = L.KW_QUEUE_SYNC
    Async = L.KW_QUEUE_ASYNC


class TaskState(enum.Enum):
    Pending = L.KW_TASK_PENDING
    Running = L.KW_TASK_RUNNING
    Done = L.KW_TASK_DONE
    Failed = L.KW_TASK_FAILED


class TaskHandle:
    def __init__(self, ev: Optional[int], failed: Optional[Exception] = None):
        self._ev = ev
        self._failed = failed

    def state(self) -> TaskState:
        if self._failed is not None:
            return TaskState.Failed
        if self._ev is None:  # a Sync queue's task: complete when enqueue returned
            return TaskState.Done
        s = C.c_int()
        _raise_for(L.lib().kw_event_state(self._ev, C.byref(s)))
        return TaskState(s.value)

    def error(self):
        return self._failed if self.state() == TaskState.Failed else None

    def __del__(self):
        if self._ev:
            try:
                L.lib().kw_event_destroy(self._ev)
            except Exception:
                pass


@dataclass
class ExecTask:
    backend: BackendKind
    workDiv: WorkDiv
    body: Callable[["Queue"], int]


@dataclass
class CopyTask:
    body: Callable[["Queue"], int]


class Queue:
    """In-order FIFO bound to one GPU: a CUDA stream. Sync completes each task inside
    enqueue; Async returns immediately. wait() raises TaskError for failures since the last
    report (queue.hpp:86-137)."""

    def __init__(self, device: Device, flavor: QueueFlavor):
        if device.isHost():
            raise UsageError("Queue: the B200 build runs queues on a GPU device (Device.gpu(i))")
        h = C.c_void_p()
        _raise_for(L.lib().kw_queue_create(device.cuda_index(), flavor.value, C.byref(h)))
        self._h = h.value
        self._device = device
        self._flavor = flavor
        self._lock = threading.Lock()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                L.lib().kw_queue_destroy(h)
            except Exception:
                pass
            self._h = None

    def handle(self) -> int:
        return self._h

    def device(self) -> Device:
        return self._device

    def flavor(self) -> QueueFlavor:
        return self._flavor

    def enqueue(self, task) -> TaskHandle:
        with self._lock:
            st = task.body(self)
            if st == L.KW_USAGE:
                _raise_for(st)  # preconditions fail before anything is enqueued
            if st == L.KW_RESOURCE:
                _raise_for(st)
            failed = TaskError(1, L.last_error()) if st == L.KW_TASK else None
            if self._flavor == QueueFlavor.Sync:  # completed inside the call: no event needed
                return TaskHandle(None, failed)
            ev = C.c_void_p()
            if L.lib().kw_task_marker(self._h, C.byref(ev)) != L.KW_OK:
                return TaskHandle(None, TaskError(1, L.last_error()))
            return TaskHandle(ev.value, failed)

    def wait(self) -> None:
        _raise_for(L.lib().kw_queue_wait(self._h))

    def report(self) -> None:
        """Sync queues: raise TaskError for failures since the last report, without a stream
        round trip (the tasks completed inside enqueue)."""
        _raise_for(L.lib().kw_queue_report(self._h))

    def shutdown(self) -> None:
        _raise_for(L.lib().kw_queue_shutdown(self._h))


_default_queues: dict = {}


def _default_queue(device: Device) -> Queue:
    dev = device if not device.isHost() else Device.gpu(0)
    q = _default_queues.get(dev.index())
    if q is None:
        q = Queue(dev, QueueFlavor.Sync)
        _default_queues[dev.index()] = q
    return q


def createCopy(dst: Buffer, src: Buffer, extent: IndexVec) -> CopyTask:
    """buffer.cpp:99-146: validated here, before anything is enqueued."""
    if dst.dim() != src.dim() or dst.dim() != extent.dim():
        raise UsageError("copy: buffer and extent dimensionalities must match")
    if dst.elemSize() != src.elemSize():
        raise UsageError("copy: element sizes must match")
    for k in range(extent.dim()):
        if extent[k] > dst.extent()[k] or extent[k] > src.extent()[k]:
            raise UsageError("copy: extent exceeds a buffer extent")
    d = (dst.data(), dst.rowPitch(), L.sz3(dst.extent().tuple()))
    s = (src.data(), src.rowPitch(), L.sz3(src.extent().tuple()))
    ext = L.sz3(extent.tuple())
    dim, es = extent.dim(), dst.elemSize()
    keep = (dst, src)

    def body(q: Queue, _keep=keep) -> int:
        return L.lib().kw_copy(q.handle(), d[0], d[1], d[2], s[0], s[1], s[2], dim, ext, es)

    return CopyTask(body)


def copyBuffer(q: Queue, dst: Buffer, src: Buffer, extent: IndexVec) -> TaskHandle:
    return q.enqueue(createCopy(dst, src, extent))


# ---- matrix CSV (buffer_csv.hpp; the text of the reference's writer, "%.17g" per value) ----------
def writeBufferCsv(buf: Buffer, stream) -> None:
    """One line per row, ',' between values; 2-D double buffers only (GPU buffers are read back)."""
    if buf.dim() != 2:
        raise UsageError("writeBufferCsv: only 2-D buffers are supported")
    if buf.elemSize() != 8:
        raise UsageError("writeBufferCsv: only double elements are supported")
    for row in buf.download():
        stream.write(",".join("%.17g" % v for v in row) + "\n")


def readBufferCsv(stream, device: Optional[Device] = None) -> Buffer:
    """Parses a CSV matrix into a new 2-D double buffer; ragged, empty or malformed input is a
    UsageError (buffer_csv.cpp semantics: a final newline ends the input)."""
    rows = []
    for line in stream.read().split("\n"):
        rows.append(line)
    if rows and rows[-1] == "":
        rows.pop()
    values = []
    for line in rows:
        line = line.rstrip("\r")
        try:
            vals = [float(t) for t in line.split(",")]
        except ValueError:
            raise UsageError(f"readBufferCsv: malformed number in '{line}'") from None
        if values and len(vals) != len(values[0]):
            raise UsageError("readBufferCsv: ragged rows")
        values.append(vals)
    if not values or not values[0]:
        raise UsageError("readBufferCsv: empty input")
    arr = np.asarray(values, dtype=np.float64)
    out = Buffer(device or Device.host(), IndexVec(*arr.shape), 8)
    if out.device().isHost():
        out.host_view()[:, : arr.shape[1]] = arr
    else:
        out.upload(arr)
    return out


# ---- kernels (kernels/axpy.hpp, kernels/gemm.hpp) ----------------------------------------------
@dataclass
class AxpyArgs:
    n: int = 0
    alpha: float = 0.0
    x: Optional[Buffer] = None
    y: Optional[Buffer] = None


@dataclass
class GemmArgs:
    m: int = 0
    n: int = 0
    k: int = 0
    alpha: float = 0.0
    beta: float = 0.0
    a: Optional[Buffer] = None
    b: Optional[Buffer] = None
    c: Optional[Buffer] = None
    tile: int = 128
    bitwise: bool = False  # tiled kernel in bit-exact mode (separately rounded, ascending k)


class AxpyKernel:
    """Y <- alpha*X + Y, bit-exact vs axpyReference (kernels/axpy.hpp:20-26)."""

    def bind(self, wd: WorkDiv, args: AxpyArgs) -> Callable[[Queue], int]:
        if args.x is None or args.y is None:
            raise UsageError("AxpyArgs: null buffer")
        if args.x.elemSize() != args.y.elemSize() or args.x.elemSize() not in (4, 8):
            raise UsageError("Buffer: typed access with mismatching element size")
        if args.n > args.x.extent().product() or args.n > args.y.extent().product():
            raise UsageError("axpy: n exceeds a buffer extent")
        cwd = wd.to_c()
        f = L.lib().kw_axpy_f32 if args.x.elemSize() == 4 else L.lib().kw_axpy_f64
        xp, yp, n, a = args.x.data(), args.y.data(), int(args.n), float(args.alpha)
        keep = (args.x, args.y)
        return lambda q, _k=keep: f(q.handle(), C.byref(cwd), n, a, xp, yp)


class GemmTiledKernel:
    """C <- alpha*A*B + beta*C, FP64 DMMA tensor cores (kernels/gemm.hpp:103-115)."""

    naive = False

    def bind(self, wd: WorkDiv, args: GemmArgs) -> Callable[[Queue], int]:
        for nm in ("a", "b", "c"):
            bf = getattr(args, nm)
            if bf is None:
                raise UsageError(f"GemmArgs: null {nm}")
            if bf.elemSize() != 8 or bf.dim() != 2:
                raise UsageError("Buffer: typed access with mismatching element size")
        a, b, c = args.a, args.b, args.c
        if args.k > 0 and (a.extent()[0] < args.m or a.extent()[1] < args.k or b.extent()[0] < args.k
                           or b.extent()[1] < args.n):
            raise UsageError("gemm: extents exceed a buffer extent")
        if c.extent()[0] < args.m or c.extent()[1] < args.n:
            raise UsageError("gemm: extents exceed a buffer extent")
        cwd = wd.to_c()
        if self.naive:
            f = L.lib().kw_dgemm_naive
        else:
            f = L.lib().kw_dgemm_bitwise if args.bitwise else L.lib().kw_dgemm
        vals = (int(args.m), int(args.n), int(args.k), float(args.alpha), a.data(), a.leadingDim(), b.data(),
                b.leadingDim(), float(args.beta), c.data(), c.leadingDim())
        keep = (a, b, c)
        return lambda q, _k=keep: f(q.handle(), C.byref(cwd), *vals)


class GemmNaiveKernel(GemmTiledKernel):
    """GemmNaiveKernel (kernels/gemm.hpp:94-101): bitwise identical to gemmReference."""

    naive = True


def axpyWorkDiv(backend: BackendKind, n: int, threadsPerBlock: int, elementsPerThread: int) -> WorkDiv:
    return divideForBackend(IndexVec(n), backend, IndexVec(threadsPerBlock), IndexVec(elementsPerThread))


def gemmNaiveWorkDiv(backend: BackendKind, m: int, n: int, threadsPerBlock: int, elementsPerThread: int) -> WorkDiv:
    return divideForBackend(IndexVec(m, n), backend, IndexVec(threadsPerBlock, 1), IndexVec(1, elementsPerThread))


def gemmTiledWorkDiv(backend: BackendKind, m: int, n: int, tile: int) -> WorkDiv:
    """gemm.cpp:127-135; on GpuCudaRt the tile is one of the DMMA kernel's tiles (64, 128)."""
    if tile == 0:
        raise UsageError("gemmTiledWorkDiv: tile edge must be positive")
    blocks = IndexVec((m + tile - 1) // tile, (n + tile - 1) // tile)
    if backend == BackendKind.GpuCudaRt:
        wd = L.kw_workdiv()
        _raise_for(L.lib().kw_dgemm_default_workdiv(m, n, tile, C.byref(wd)))
        return WorkDiv.from_c(wd)
    if backend == BackendKind.ThreadsParallel:
        return WorkDiv(blocks, IndexVec(tile, 1), IndexVec(1, tile))
    return WorkDiv(blocks, IndexVec(1, 1), IndexVec(tile, tile))


def createExec(backend: BackendKind, wd: WorkDiv, kernel, *args) -> ExecTask:
    """queue.hpp:74-82: binds backend, division, kernel and args (validated now)."""
    if backend != BackendKind.GpuCudaRt:
        raise UsageError(f"createExec: back-end '{backendName(backend)}' does not exist in the B200 build "
                         "(no CPU fallback); use BackendKind.GpuCudaRt")
    if len(args) != 1:
        raise UsageError("createExec: kernels take exactly one argument struct")
    return ExecTask(backend, wd, kernel.bind(wd, args[0]))


def executeTask(backend: BackendKind, wd: WorkDiv, kernel, *args) -> None:
    """exec.hpp:32-36: externally synchronous run on the device of the output buffer."""
    task = createExec(backend, wd, kernel, *args)
    out = args[0].y if isinstance(args[0], AxpyArgs) else args[0].c
    q = _default_queue(out.device())
    q.enqueue(task)
    q.report()
