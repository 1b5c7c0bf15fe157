#!/usr/bin/env python
"""bench.py — the kernelweave B200 hot path on BASELINE.json's configs.

Headline (the JSON line's metric/value): AXPY fp32, n = 2^28 (BASELINE.json configs[1]), inputs
resident in HBM, index-sharded across ranks under torchrun (strong scaling: total n fixed).
The same line carries:
  e2e          the same metric through the public API with host (pinned) buffers: H2D of X, Y
               and D2H of Y inside the timed region (Queue.enqueue + wait, like runner.cpp:114-117);
               each rank streams only its own shard, pinned on its GPU's NUMA node
  roofline     AXPY kernel vs MEASURED_PEAKS.json hbm_gbs (algorithmic 12 B/element); `kernel` is
               the template the launch runs (kw_axpy_kernel_name)
  cpu_baseline the reference's own CPU AXPY (oracle/_ref: reference runtime, BlocksParallel,
               all host cores) on the same global input, rank 0, at every N
  parity       at every N: each rank's GPU Y digest after the first step and after all
               1 + W + K steps vs the reference CPU Y over the same index range
  dgemm        DGEMM fp64 TFLOP/s: 8192^3 (north-star headline) and 4096^3 (configured point)
               at N = 1; 16384^3 row-block sharded with NCCL broadcast of B at N > 1, with
               sampled-row parity (CPU reference + 1-GPU kw_dgemm) and a CPU baseline
  clocks, gpu_launches

`--impl reference` runs only the reference CPU implementation (rank 0) on the same config,
--warmup + --steps runs.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_AXPY = 1 << 28
BYTES_PER_ELEM = 12  # read X, read Y, write Y (fp32)
FP64_NOMINAL_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12  # 37.2: 148 SMs x 64 FP64 FMA/clk x 1.965 GHz


INPUT_BLOCK = 1 << 20  # elements per independently seeded block of the synthetic AXPY input
AXPY_DATA = (f"synthetic (numpy U[0,10), {INPUT_BLOCK}-element blocks seeded [1234, block]; identical global "
             f"input at every N, each rank generates only its shard)")
DGEMM_PEAK_PROBE = 37.16  # DMMA throughput measured on this pool (tools/probe/probe.cu)


def axpy_config(world: int, tpb: int, ept: int) -> dict:
    """The headline's `config` — built from the arguments alone, so both arms print it identically."""
    from paper_1602_08477_b200 import sharding as S
    lo, hi = S.axpy_range(N_AXPY, world, 0)
    n = hi - lo
    return {"workload": "AXPY fp32 n=2^28 index-sharded (BASELINE.json configs[1])", "n": N_AXPY,
            "n_per_rank": n, "workdiv": {"threads": tpb, "elems": ept, "blocks": -(-n // (tpb * ept))},
            "parallelism": f"index-shard x{world} (no collective)",
            "l2": "inputs larger than L2 (2.15 GB read+write per step vs 132 MB L2); no flush needed"}


def axpy_inputs(lo: int, hi: int, seed: int = 1234, out=None):
    """X, Y over [lo, hi) of the global synthetic input, U[0,10) fp32. The global input is cut into
    INPUT_BLOCK-element blocks, block b drawn (X then Y) from default_rng([seed, b]): a rank
    generates only its own shard, and every rank count sees the same global bytes."""
    n = hi - lo
    x, y = out if out is not None else (np.empty(n, np.float32), np.empty(n, np.float32))
    ten = np.float32(10)
    for b in range(lo // INPUT_BLOCK, -(-hi // INPUT_BLOCK)):
        g = np.random.default_rng([seed, b])
        bx = g.random(INPUT_BLOCK, dtype=np.float32) * ten
        by = g.random(INPUT_BLOCK, dtype=np.float32) * ten
        s0, s1 = max(lo, b * INPUT_BLOCK), min(hi, (b + 1) * INPUT_BLOCK)
        x[s0 - lo:s1 - lo] = bx[s0 - b * INPUT_BLOCK:s1 - b * INPUT_BLOCK]
        y[s0 - lo:s1 - lo] = by[s0 - b * INPUT_BLOCK:s1 - b * INPUT_BLOCK]
    return x, y


def gemm_rows(seed: int, rows, cols: int) -> np.ndarray:
    """Rows of a synthetic U[0,10) fp64 matrix, row r drawn from default_rng([seed, r]): any rank
    (or the checker on rank 0) can regenerate any row without the rest of the matrix."""
    rows = list(rows)
    out = np.empty((len(rows), cols))
    for i, r in enumerate(rows):
        out[i] = np.random.default_rng([seed, r]).random(cols) * 10
    return out


def digest(a: np.ndarray) -> str:
    import hashlib
    return hashlib.blake2b(np.ascontiguousarray(a), digest_size=16).hexdigest()


def numa_node_of(lib, device: int):
    """(node, cpus) the GPU's PCIe root sits on (sysfs), or None when unknown."""
    buf = C.create_string_buffer(64)
    if lib.kw_device_pci_bus_id(device, buf, 64) != 0:
        return None
    try:
        node = int(Path(f"/sys/bus/pci/devices/{buf.value.decode()}/numa_node").read_text())
        if node < 0:
            return None
        cpus = set()
        for part in Path(f"/sys/devices/system/node/node{node}/cpulist").read_text().strip().split(","):
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
        cpus &= os.sched_getaffinity(0)
        return (node, cpus) if cpus else None
    except (OSError, ValueError):
        return None


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("hbm_gbs", 6650.0), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def traffic_from_profiles(kernel: str):
    """dram bytes per launch from the committed ncu --set full summary, or None."""
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        d = json.loads(p.read_text())
        v = d.get(kernel)
        if isinstance(v, dict):
            return v.get("dram_bytes_per_launch")
    return None


class ClockSampler:
    """nvidia-smi samples (200 ms..50 ms period) during the timed regions."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.active = False
        self.samples = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-i", str(self.gpu), "-lms", "50"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None
            return
        threading.Thread(target=self._reader, daemon=True).start()

    def _reader(self):
        for line in self.proc.stdout:
            if self.active:
                self.samples.append(line.strip())

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for s in self.samples:
            f = [x.strip() for x in s.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------------------------------
# distributed plumbing
# --------------------------------------------------------------------------------------------
class Dist:
    def __init__(self, n_gpus: int, backend: str = "nccl", same_gpu: bool = False):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        # --same-gpu (gloo only): every rank on GPU 0 — a harness self-test of the N > 1 code path
        # on a one-GPU box; ranks never wait on one another inside a kernel.
        self.local = 0 if same_gpu else int(os.environ.get("LOCAL_RANK", "0"))
        self.backend = backend
        self.pg = None
        if self.world > 1:
            import torch
            import torch.distributed as dist
            if torch.cuda.is_available():
                torch.cuda.set_device(self.local)
            if backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            else:
                dist.init_process_group("gloo")
            self.dist = dist
            self.torch = torch
        if n_gpus != self.world and self.rank == 0:
            print(f"warning: --gpus {n_gpus} but WORLD_SIZE={self.world}", file=sys.stderr)

    def _dev(self):
        return "cuda" if self.backend == "nccl" else "cpu"

    def barrier(self):
        if self.world > 1:
            if self.backend == "nccl":
                self.dist.barrier(device_ids=[self.local])
            else:
                self.dist.barrier()

    def quiet_wait_for_rank0(self, key: str):
        """Ranks > 0 block in the rendezvous store (a socket wait, no spinning host thread) until
        rank 0 calls it with the same key after its CPU-side work — so the CPU baseline rank 0
        times is not competing with N - 1 ranks spinning in a collective on the same host."""
        if self.world == 1:
            return
        store = self.dist.distributed_c10d._get_default_store()
        if self.rank == 0:
            store.set(key, "1")
        else:
            import datetime
            store.wait([key], datetime.timedelta(seconds=1800))
        self.barrier()

    def max(self, v: float) -> float:
        if self.world == 1:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device=self._dev())
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, v: float) -> float:
        if self.world == 1:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device=self._dev())
        self.dist.all_reduce(t)
        return float(t.item())

    def gather_objects(self, obj) -> list:
        """Every rank's `obj`, in rank order, on every rank (test/parity plumbing only)."""
        if self.world == 1:
            return [obj]
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out

    def bcast_bytes(self, b: bytes | None) -> bytes:
        if self.world == 1:
            return b
        obj = [b]
        self.dist.broadcast_object_list(obj, src=0)
        return obj[0]

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


# --------------------------------------------------------------------------------------------
# product arm
# --------------------------------------------------------------------------------------------
def run_ours(args, dist: Dist) -> dict:
    from paper_1602_08477_b200 import _lib as L
    from paper_1602_08477_b200 import kernelweave as kw

    lib = L.lib()
    dev = kw.Device.gpu(dist.local)
    gpu_index = dist.local
    GPU = kw.BackendKind.GpuCudaRt
    q = kw.Queue(dev, kw.QueueFlavor.Async)

    from paper_1602_08477_b200 import sharding as S
    lo, hi = S.axpy_range(N_AXPY, dist.world, dist.rank)
    n = hi - lo
    alpha = np.float32(9.096465)
    # This rank's pinned host shard, allocated and first-touched from the GPU's NUMA node (each
    # rank streams over its own PCIe link; remote-node pinned pages would cross the socket link).
    numa = numa_node_of(lib, gpu_index)
    affinity = os.sched_getaffinity(0)
    if numa:
        os.sched_setaffinity(0, numa[1])
    try:
        hx = kw.Buffer(kw.Device.host(), kw.IndexVec(n), 4)
        hy = kw.Buffer(kw.Device.host(), kw.IndexVec(n), 4)
        xs, ys = axpy_inputs(lo, hi, out=(hx.host_view(), hy.host_view()))
    finally:
        os.sched_setaffinity(0, affinity)

    x = kw.Buffer(dev, kw.IndexVec(n), 4)
    y = kw.Buffer(dev, kw.IndexVec(n), 4)
    x.upload(xs)
    y.upload(ys)
    wd = kw.axpyWorkDiv(GPU, n, args.tpb, args.ept)
    task = kw.createExec(GPU, wd, kw.AxpyKernel(), kw.AxpyArgs(n, float(alpha), x, y))
    wdc = wd.to_c()
    kname = C.create_string_buffer(96)
    L.check(lib.kw_axpy_kernel_name(C.byref(wdc), 4, x.data(), y.data(), kname, 96))

    # Parity: Y after the first step (from pristine inputs) and after all 1 + W + K steps are
    # hashed per rank; rank 0 checks both against the reference CPU run on the global input.
    q.enqueue(task)
    q.wait()
    dig_first = digest(y.download())

    sampler = ClockSampler(gpu_index)
    sampler.start()
    time.sleep(0.3)

    # The timed loop calls the C-ABI entry point (kw_axpy_f32: the same kernel and division as
    # `task`): a TaskHandle per enqueue would put an event between consecutive kernels, which
    # both costs an event per step and stops programmatic dependent launch from overlapping one
    # step's launch with the previous step's tail.

    def step():
        L.check(lib.kw_axpy_f32(q.handle(), C.byref(wdc), n, float(alpha), x.data(), y.data()))

    for _ in range(args.warmup):
        step()
    q.wait()
    evs = []

    def rec():
        ev = C.c_void_p()
        L.check(lib.kw_event_record(q.handle(), C.byref(ev)))
        return ev

    dist.barrier()
    q.wait()
    launches0 = lib.kw_launch_count()
    sampler.active = True
    evs.append(rec())
    for _ in range(args.steps):
        step()
    evs.append(rec())
    q.wait()
    dist.barrier()
    sampler.active = False
    launches = lib.kw_launch_count() - launches0
    ms = C.c_float()
    L.check(lib.kw_event_elapsed_ms(evs[0], evs[1], C.byref(ms)))
    for e in evs:
        lib.kw_event_destroy(e)
    per = [ms.value / args.steps]
    local_ms = ms.value
    total_ms = dist.max(local_ms)
    total_bytes = BYTES_PER_ELEM * N_AXPY * args.steps
    value = total_bytes / (total_ms / 1e3) / 1e9
    peak, peak_src = peaks()
    achieved = BYTES_PER_ELEM * n / (statistics.mean(per) / 1e3) / 1e9
    dig_final = digest(y.download())
    applied = 1 + args.warmup + args.steps
    del x, y

    # ---- e2e: host (pinned) buffers through the public API, copies inside the timed region
    e2e_steps = max(3, min(args.e2e_steps, args.steps))
    htask = kw.createExec(GPU, wd, kw.AxpyKernel(), kw.AxpyArgs(n, float(alpha), hx, hy))
    for _ in range(2):  # first host-buffer passes on a fresh box run slow (page state); keep them untimed
        q.enqueue(htask)
        q.wait()
    dist.barrier()
    sampler.active = True
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        q.enqueue(htask)
        q.wait()
    t1 = time.perf_counter()
    sampler.active = False
    e2e_local = t1 - t0
    e2e_s = dist.max(e2e_local)
    e2e_value = BYTES_PER_ELEM * N_AXPY * e2e_steps / e2e_s / 1e9
    rank_link = BYTES_PER_ELEM * n * e2e_steps / e2e_local / 1e9
    del hx, hy, xs, ys

    # ---- fp64 AXPY (the reference's own AxpyKernel dtype), same n, device-resident
    f64 = None
    if not args.no_f64:
        x64 = kw.Buffer(dev, kw.IndexVec(n), 8)
        y64 = kw.Buffer(dev, kw.IndexVec(n), 8)
        L.check(lib.kw_memset(q.handle(), x64.data(), 0, n * 8))
        L.check(lib.kw_memset(q.handle(), y64.data(), 0, n * 8))
        wd64 = kw.axpyWorkDiv(GPU, n, args.tpb, max(2, args.ept // 2)).to_c()

        def step64():  # C-ABI per step, as in the fp32 loop above
            L.check(lib.kw_axpy_f64(q.handle(), C.byref(wd64), n, 1.5, x64.data(), y64.data()))

        for _ in range(3):
            step64()
        q.wait()
        dist.barrier()
        a64, b64 = C.c_void_p(), C.c_void_p()
        steps64 = max(10, args.steps // 4)
        L.check(lib.kw_event_record(q.handle(), C.byref(a64)))
        for _ in range(steps64):
            step64()
        L.check(lib.kw_event_record(q.handle(), C.byref(b64)))
        q.wait()
        ms64 = C.c_float()
        L.check(lib.kw_event_elapsed_ms(a64, b64, C.byref(ms64)))
        lib.kw_event_destroy(a64)
        lib.kw_event_destroy(b64)
        t = dist.max(ms64.value)
        f64 = {"value": round(24 * N_AXPY * steps64 / (t / 1e3) / 1e9, 1), "unit": "GB/s", "steps": steps64,
               "bytes_per_elem": 24, "note": "AXPY fp64 n=2^28 (the reference's AxpyKernel dtype), HBM-resident"}
        del x64, y64

    gathered = dist.gather_objects((lo, hi, dig_first, dig_final, round(rank_link, 2), numa[0] if numa else None))
    out = {
        "metric": "AXPY fp32 HBM GB/s (n=2^28, Y=alpha*X+Y, 12 B/elem)",
        "value": round(value, 1),
        "unit": "GB/s",
        "n_gpus": dist.world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(total_ms / args.steps, 5),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32",
        "data": AXPY_DATA,
        "config": axpy_config(dist.world, args.tpb, args.ept),
        "e2e": {"value": round(e2e_value, 2), "unit": "GB/s", "steps": e2e_steps,
                "h2d_bytes_per_step": 8 * N_AXPY, "d2h_bytes_per_step": 4 * N_AXPY,
                "how": "executeTask-equivalent Queue.enqueue(createExec(GpuCudaRt, AxpyKernel, host pinned "
                       "buffers)) + wait, wall clock, max over ranks; each rank streams its own shard over its "
                       "own PCIe link from pinned pages placed on the GPU's NUMA node; chunked H2D/kernel/D2H "
                       "on three streams",
                "per_rank_link_gbs": [g[4] for g in gathered] if gathered else None,
                "numa_nodes": [g[5] for g in gathered] if gathered else None,
                "link_ceiling": {"value": round(78.8 * dist.world, 1), "per_rank": 78.8, "unit": "GB/s",
                                 "what": "pure pinned copies with the same 2:1 H2D:D2H byte mix, one link per "
                                         "GPU (x N ranks)",
                                 "source": "profiles/pcie_probe_r01.txt"}},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "peak_source": peak_src,
                     "traffic": (None if traffic_from_profiles("axpy_f32") is None
                                 else round(traffic_from_profiles("axpy_f32") * n / N_AXPY)),
                     "traffic_source": "profiles/traffic.json (ncu --set full at n=2^28, scaled to this rank's "
                                       "shard)",
                     "kernel": kname.value.decode(), "bytes_per_launch": BYTES_PER_ELEM * n},
        "gpu_launches": int(launches),
        "clocks": None,
        "axpy_f64": f64,
        "dgemm": None,
    }

    if dist.rank == 0 and not args.no_cpu:
        cb, parity = cpu_baseline_axpy(alpha, gathered, applied, args.warmup)
        out["cpu_baseline"] = cb
        out["parity"] = parity
    dist.quiet_wait_for_rank0("kw-axpy-cpu-baseline-done")  # rank 0 ran the CPU reference meanwhile

    # ---- secondary: DGEMM. Guarded: neither an exception nor a hang in this leg (an N > 1
    # communicator that never forms, say) may cost the headline line above — a watchdog prints
    # the line with the DGEMM leg marked failed and ends the rank.
    def on_timeout():
        if dist.rank == 0:
            partial = dict(out)
            partial["dgemm"] = {"error": f"DGEMM leg exceeded {args.dgemm_timeout:.0f} s on some rank; skipped"}
            partial["clocks"] = sampler.summary()
            print(json.dumps(partial), flush=True)
        os._exit(0)

    watchdog = threading.Timer(args.dgemm_timeout, on_timeout)
    watchdog.daemon = True
    watchdog.start()
    try:
        dg = run_dgemm(args, dist, kw, L, lib, dev, q, sampler)
    except Exception as ex:  # reported in the line, not fatal to it
        dg = {"error": f"{type(ex).__name__}: {str(ex)[:300]}"}
    finally:
        watchdog.cancel()
    sampler.stop()
    out["clocks"] = sampler.summary()
    out["dgemm"] = dg
    return out


def run_dgemm(args, dist, kw, L, lib, dev, q, sampler) -> dict:
    """DGEMM fp64: N = 1 -> 8192^3 (headline) + 4096^3; N > 1 -> 16384^3 row-sharded with NCCL
    broadcast of B in column panels (kw_dgemm_rowsharded)."""
    if args.no_dgemm:
        return None
    GPU = kw.BackendKind.GpuCudaRt
    res = {"metric": "DGEMM fp64 TFLOP/s (2*M*N*K)", "unit": "TFLOP/s",
           "peak_nominal_tflops": round(FP64_NOMINAL_TFLOPS, 2),
           "peak_source": "nominal 148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz (DMMA measured 37.16 TF on this "
                          "pool: tools/probe/probe.cu)"}

    def timed(fn, steps, warm=2):
        for _ in range(warm):
            fn()
        q.wait()
        dist.barrier()
        a, b = C.c_void_p(), C.c_void_p()
        sampler.active = True
        L.check(lib.kw_event_record(q.handle(), C.byref(a)))
        for _ in range(steps):
            fn()
        L.check(lib.kw_event_record(q.handle(), C.byref(b)))
        q.wait()
        sampler.active = False
        ms = C.c_float()
        L.check(lib.kw_event_elapsed_ms(a, b, C.byref(ms)))
        lib.kw_event_destroy(a)
        lib.kw_event_destroy(b)
        dist.barrier()
        return dist.max(ms.value)

    rng = np.random.default_rng(77)
    if dist.world == 1 and not args.force_rowsharded:
        for size, steps in ((8192, args.dgemm_steps), (4096, args.dgemm_steps * 4)):
            a = rng.random((size, size)) * 10
            b = rng.random((size, size)) * 10
            c = rng.random((size, size)) * 10
            A, B, Cb = (kw.Buffer(dev, kw.IndexVec(size, size), 8) for _ in range(3))
            A.upload(a)
            B.upload(b)
            Cb.upload(c)
            task = kw.createExec(GPU, kw.gemmTiledWorkDiv(GPU, size, size, 128), kw.GemmTiledKernel(),
                                 kw.GemmArgs(size, size, size, 1.25, 0.75, A, B, Cb))
            ms = timed(lambda: q.enqueue(task), steps)
            tflops = 2 * size ** 3 * steps / (ms / 1e3) / 1e12
            entry = {"value": round(tflops, 3), "ms_per_step": round(ms / steps, 4), "steps": steps,
                     "roofline": {"bound": "fp64", "achieved": round(tflops, 3),
                                  "peak": round(FP64_NOMINAL_TFLOPS, 2), "unit": "TFLOP/s",
                                  "frac": round(tflops / FP64_NOMINAL_TFLOPS, 4),
                                  "peak_source": "nominal (148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz)",
                                  "peak_dmma_probe": DGEMM_PEAK_PROBE,
                                  "frac_of_dmma_probe": round(tflops / DGEMM_PEAK_PROBE, 4),
                                  "traffic": traffic_from_profiles(f"dgemm_{size}")}}
            # e2e: host pinned buffers, H2D of A, B, C and D2H of C per step
            hA, hB, hC = (kw.Buffer(kw.Device.host(), kw.IndexVec(size, size), 8) for _ in range(3))
            for hb, src in ((hA, a), (hB, b), (hC, c)):
                hb.host_view()[:, :size] = src
            htask = kw.createExec(GPU, kw.gemmTiledWorkDiv(GPU, size, size, 128), kw.GemmTiledKernel(),
                                  kw.GemmArgs(size, size, size, 1.25, 0.75, hA, hB, hC))
            for _ in range(2):  # untimed host passes (first passes on a fresh box run slow)
                q.enqueue(htask)
                q.wait()
            e2e_steps = 8
            sampler.active = True
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                q.enqueue(htask)
                q.wait()
            e2e_s = time.perf_counter() - t0
            sampler.active = False
            # the library's schedule choice (kw_dgemm.cu dgemm_streamed): >= 400 flop/B -> streamed
            intensity = 2 * size ** 3 / (8 * 3 * size * size)
            streamed = intensity >= float(os.environ.get("KW_E2E_MIN_INTENSITY", "400")) and \
                os.environ.get("KW_E2E_STREAMED", "1") != "0"
            entry["e2e"] = {"value": round(2 * size ** 3 * e2e_steps / e2e_s / 1e12, 3), "unit": "TFLOP/s",
                            "steps": e2e_steps, "h2d_bytes_per_step": 3 * size * size * 8,
                            "d2h_bytes_per_step": size * size * 8,
                            "schedule": ("streamed: square-growth panel uploads into one persistent kernel, "
                                          "k split 1/4 + 3/4 (first pass on the first quarter of A/B)"
                                         if streamed else "row panels of A/C, B streamed in column panels")}
            bw_task = None
            if size == 8192:
                # bit-exact tiled mode: separately rounded products/sums in ascending k
                bw_task = kw.createExec(GPU, kw.gemmTiledWorkDiv(GPU, size, size, 128), kw.GemmTiledKernel(),
                                        kw.GemmArgs(size, size, size, 1.25, 0.75, A, B, Cb, 128, bitwise=True))
                bsteps = max(2, steps // 3)
                bms = timed(lambda: q.enqueue(bw_task), bsteps, warm=1)
                entry["bitwise_mode"] = {"value": round(2 * size ** 3 * bsteps / (bms / 1e3) / 1e12, 3),
                                         "unit": "TFLOP/s", "steps": bsteps,
                                         "note": "GemmTiledKernel bitwise=True: DMUL+DADD in ascending k, "
                                                 "bitwise equal to gemmReference (FP64-pipe bound)"}
            if size == 8192 and not args.no_cpu:
                entry["cpu_baseline"], entry["parity"] = cpu_baseline_dgemm(a, b, c, 1.25, 0.75, Cb, q, task, bw_task)
            res[f"n{size}"] = entry
            del A, B, Cb, hA, hB, hC
        # the small end of the BASELINE configs[4] sweep (the library's own tile choice)
        sweep = {}
        for size in (1024, 2048):
            a = rng.random((size, size)) * 10
            A, B, Cb = (kw.Buffer(dev, kw.IndexVec(size, size), 8) for _ in range(3))
            for buf in (A, B, Cb):
                buf.upload(a)
            task = kw.createExec(GPU, kw.gemmTiledWorkDiv(GPU, size, size, 128), kw.GemmTiledKernel(),
                                 kw.GemmArgs(size, size, size, 1.25, 0.75, A, B, Cb))
            steps = max(20, int(2e12 / (2 * size ** 3)))
            ms = timed(lambda: q.enqueue(task), steps)
            tflops = 2 * size ** 3 * steps / (ms / 1e3) / 1e12
            sweep[f"n{size}"] = {"value": round(tflops, 3), "steps": steps, "unit": "TFLOP/s",
                                 "frac": round(tflops / FP64_NOMINAL_TFLOPS, 4),
                                 "frac_of_dmma_probe": round(tflops / DGEMM_PEAK_PROBE, 4),
                                 "traffic": traffic_from_profiles(f"dgemm_{size}")}
            del A, B, Cb
        res["sweep"] = sweep
        if not args.no_cublas:
            res["cublas_same_box"] = cublas_dgemm(dist.local, (8192, 4096, 2048, 1024))
        res["value"] = res["n8192"]["value"]
        res["config"] = "DGEMM fp64 M=N=K=8192 (north-star headline) and 4096 (BASELINE configs[2]), 1 GPU"
        return res

    # N > 1: 16384^3, A/C row blocks per rank, B broadcast from rank 0 in column panels.
    if args.same_gpu:
        # NCCL refuses two ranks on one GPU: the --same-gpu harness self-test covers the AXPY
        # shards and timing reductions only (the panel pipeline has --force-rowsharded).
        return {"skipped": "--same-gpu self-test: NCCL needs one GPU per rank (see --force-rowsharded)"}
    return run_dgemm_rowsharded(args, dist, kw, L, lib, dev, q, timed, res)


def run_dgemm_rowsharded(args, dist, kw, L, lib, dev, q, timed, res) -> dict:
    """16384^3 row-sharded: rank r owns rows [r0, r1) of A and C, rank 0 owns B; each step is one
    kw_dgemm_rowsharded (ncclBroadcast of B in column panels overlapped with the panel DGEMMs).
    Parity at every N (the reference verifies every measured point, runner.cpp:120-125): one step
    from pristine C, then 16 sampled rows per rank are gathered on rank 0 and checked (i) against
    the reference GemmTiledKernel on the CPU under |dC| <= (K+4)u|C_ref| and (ii) bitwise against
    a single-GPU kw_dgemm of the same rows."""
    from paper_1602_08477_b200 import sharding as S
    GPU = kw.BackendKind.GpuCudaRt
    size = 16384
    seed_a, seed_b, seed_c = 161, 162, 163
    alpha, beta = 1.25, 0.75
    r0, r1 = S.dgemm_rows(size, dist.world, dist.rank)
    ml = r1 - r0
    A = kw.Buffer(dev, kw.IndexVec(max(ml, 1), size), 8)
    Cb = kw.Buffer(dev, kw.IndexVec(max(ml, 1), size), 8)
    c_local = gemm_rows(seed_c, range(r0, r1), size) if ml else None
    if ml:
        A.upload(gemm_rows(seed_a, range(r0, r1), size))
        Cb.upload(c_local)
    B = None
    if dist.rank == 0:
        B = kw.Buffer(dev, kw.IndexVec(size, size), 8)
        B.upload(gemm_rows(seed_b, range(size), size))
    elems = C.c_size_t()
    L.check(lib.kw_dgemm_rowsharded_scratch(size, size, args.panels, C.byref(elems)))
    panels = kw.Buffer(dev, kw.IndexVec(elems.value), 8)
    uid = (C.c_char * 128)()
    if dist.rank == 0:
        L.check(lib.kw_comm_unique_id(uid))
    raw = dist.bcast_bytes(bytes(uid) if dist.rank == 0 else None)
    uid = (C.c_char * 128).from_buffer_copy(raw)
    comm = C.c_void_p()
    L.check(lib.kw_comm_init(C.byref(comm), dist.local, dist.world, dist.rank, uid))

    def step():
        L.check(lib.kw_dgemm_rowsharded(comm, q.handle(), ml, size, size, alpha, A.data(), A.leadingDim(),
                                        B.data() if B is not None else None,
                                        B.leadingDim() if B is not None else 0, beta, Cb.data(), Cb.leadingDim(),
                                        panels.data(), args.panels, 0))

    # parity step from pristine C: sampled rows of this rank's block
    step()
    q.wait()
    nsamp = min(16, ml)
    local_rows = [r0 + (i * ml) // nsamp for i in range(nsamp)]
    got = np.empty((nsamp, size))
    for i, r in enumerate(local_rows):
        ext = L.sz3((size,))
        L.check(lib.kw_copy(q.handle(), got[i].ctypes.data, size * 8, ext,
                            Cb.data() + (r - r0) * Cb.rowPitch(), size * 8, ext, 1, ext, 8))
    q.wait()
    del c_local
    gathered = dist.gather_objects((local_rows, got))

    steps = max(2, args.dgemm_steps // 2)
    ms = timed(step, steps, warm=1)
    lib.kw_comm_destroy(comm)
    tflops = 2 * size ** 3 * steps / (ms / 1e3) / 1e12
    per_gpu = tflops / dist.world
    res.update({"value": round(tflops, 3), "ms_per_step": round(ms / steps, 3), "steps": steps,
                "config": (f"DGEMM fp64 16384^3 row-block sharded x{dist.world}, ncclBroadcast of B in two row slabs "
                           f"(first 1/{args.panels} of the k-tiles, then the rest) overlapped with two k-range launches "
                           f"(BASELINE configs[3])" if os.environ.get("KW_ROWSHARD_SCHEDULE") != "panels" else
                           f"DGEMM fp64 16384^3 row-block sharded x{dist.world}, ncclBroadcast of B in {args.panels} "
                           f"column panels overlapped with compute (BASELINE configs[3])"),
                "roofline": {"bound": "fp64", "achieved": round(per_gpu, 3), "unit": "TFLOP/s per GPU",
                             "peak": round(FP64_NOMINAL_TFLOPS, 2), "frac": round(per_gpu / FP64_NOMINAL_TFLOPS, 4),
                             "peak_source": "nominal (148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz)",
                             "peak_dmma_probe": DGEMM_PEAK_PROBE,
                             "frac_of_dmma_probe": round(per_gpu / DGEMM_PEAK_PROBE, 4)}})
    if dist.rank == 0:
        rows = [r for rs, _ in gathered for r in rs]
        gpu_rows = np.vstack([g for _, g in gathered])
        res["cpu_baseline"], res["parity"] = dgemm_rows_check(kw, dev, q, B, rows, gpu_rows, size, alpha, beta,
                                                              (seed_a, seed_c), args.no_cpu)
    del A, Cb, B, panels
    dist.quiet_wait_for_rank0("kw-dgemm-cpu-check-done")
    return res


def dgemm_rows_check(kw, dev, q, B, rows, gpu_rows, size, alpha, beta, seeds, no_cpu):
    """Rank 0: the gathered sampled rows of the row-sharded C against (i) a single-GPU kw_dgemm
    of the same rows (bitwise: row-block invariance) and (ii) the reference GemmTiledKernel."""
    GPU = kw.BackendKind.GpuCudaRt
    a = gemm_rows(seeds[0], rows, size)
    c = gemm_rows(seeds[1], rows, size)
    R = len(rows)
    As, Cs = kw.Buffer(dev, kw.IndexVec(R, size), 8), kw.Buffer(dev, kw.IndexVec(R, size), 8)
    As.upload(a)
    Cs.upload(c)
    q.enqueue(kw.createExec(GPU, kw.gemmTiledWorkDiv(GPU, R, size, 128), kw.GemmTiledKernel(),
                            kw.GemmArgs(R, size, size, alpha, beta, As, B, Cs)))
    q.wait()
    one_gpu = Cs.download()
    parity = {"check": f"{R} rows sampled across all ranks' blocks (16 per rank): bitwise vs a 1-GPU kw_dgemm of "
                       f"the same rows, and |dC| <= (K+4)*2^-53*|C_ref| vs the reference GemmTiledKernel (CPU)",
              "rows": R, "bitwise_vs_1gpu": bool(np.array_equal(gpu_rows, one_gpu))}
    cb = None
    if not no_cpu:
        from oracle import oracle as O
        b = B.download()
        out = c.copy()
        kind = "reference" if O.ref_available() else "port"
        t = time.perf_counter()
        if kind == "reference":
            os.environ.setdefault("KERNELWEAVE_POOL_SIZE", str(cpu_threads()))
            sec = C.c_double()
            assert O.ref().kwref_gemm_kernel(1, 1, R, size, size, alpha, beta, a.ctypes.data, size, b.ctypes.data,
                                             size, out.ctypes.data, size, 32, 16, 8, C.byref(sec)) == 0
            secs = sec.value
        else:
            out = O.gemm(alpha, beta, a, b, c, threads=cpu_threads())
            secs = time.perf_counter() - t
        err = np.abs(gpu_rows - out)
        bound = (size + 4) * 2.0 ** -53 * np.abs(out)
        parity["within_tolerance"] = bool(np.all(err <= bound))
        parity["max_err_over_bound"] = round(float(np.max(err / bound)), 4)
        cb = {"value": round(2 * R * size * size / secs / 1e9, 3), "unit": "GFLOP/s", "cores": cpu_threads(),
              "kind": kind, "sample": f"{R} rows of the 16384^3 workload (GemmTiledKernel tile 32, BlocksParallel); "
                                      f"{secs:.2f} s"}
    parity["match"] = bool(parity["bitwise_vs_1gpu"] and parity.get("within_tolerance", True))
    return cb, parity


def cublas_dgemm(device: int, sizes) -> dict:
    """cuBLAS DGEMM (torch.matmul fp64) on the same box, for context only — not on our path."""
    try:
        import torch
        out = {}
        for n in sizes:
            a = torch.rand(n, n, dtype=torch.float64, device=f"cuda:{device}")
            b = torch.rand(n, n, dtype=torch.float64, device=f"cuda:{device}")
            for _ in range(2):
                a @ b
            torch.cuda.synchronize()
            reps = max(20, int(2e12 / (2 * n ** 3)))
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(reps):
                a @ b
            e1.record()
            torch.cuda.synchronize()
            out[f"n{n}"] = round(2 * n ** 3 * reps / (e0.elapsed_time(e1) / 1e3) / 1e12, 3)
            del a, b
        out["unit"] = "TFLOP/s"
        return out
    except Exception as ex:  # noqa: BLE001
        return {"error": str(ex)[:200]}


# --------------------------------------------------------------------------------------------
# CPU baseline / reference arm (the only place bench.py executes oracle/)
# --------------------------------------------------------------------------------------------
def cpu_threads():
    return len(os.sched_getaffinity(0))


def _ref_axpy_f32(xs, ys, alpha, runs, on_run=None):
    """The reference's own runtime (oracle/_ref) running the AxpyKernel functor restated for
    float on BlocksParallel with every host core, applied `runs` times in place (Y compounds,
    as the GPU's does); on_run(i, read) may read Y after run i. Returns (seconds per run, kind)."""
    from oracle import oracle as O
    n = xs.size
    times = []
    if O.ref_available():
        r = O.ref()
        os.environ.setdefault("KERNELWEAVE_POOL_SIZE", str(cpu_threads()))
        h = r.kwref_axpy_session_new(1, 1, n, float(alpha), xs.ctypes.data, ys.ctypes.data, 16, 4096)
        assert h, r.kwref_last_error()
        sec = C.c_double()
        try:
            for i in range(runs):
                assert r.kwref_axpy_session_run(h, C.byref(sec)) == 0
                times.append(sec.value)
                if on_run:
                    def read():
                        out = np.empty(n, np.float32)
                        r.kwref_axpy_session_read(h, out.ctypes.data)
                        return out
                    on_run(i, read)
        finally:
            r.kwref_axpy_session_free(h)
        return times, "reference"
    out = ys.copy()
    for i in range(runs):
        t = time.perf_counter()
        O.lib().kw_oracle_axpy_threaded(n, float(alpha), xs.ctypes.data, out.ctypes.data, 1, cpu_threads())
        times.append(time.perf_counter() - t)
        if on_run:
            on_run(i, lambda: out.copy())
    return times, "port"


def cpu_baseline_axpy(alpha, gathered, applied, warm):
    """Rank 0, every N: the reference CPU AXPY on the GLOBAL input, applied as many times as the
    GPU applied it. Its Y after the first run and after the last is hashed over each rank's
    [lo, hi) and compared with that rank's GPU digests (the reference verifies every measured
    point, runner.cpp:120-125, 264-265); its per-run time is the CPU baseline."""
    xs, ys = axpy_inputs(0, N_AXPY)
    checks = {}

    def on_run(i, read):
        if i == 0 or i == applied - 1:
            yr = read()
            checks[i] = [digest(yr[lo:hi]) for (lo, hi, *_r) in gathered]

    times, kind = _ref_axpy_f32(xs, ys, alpha, applied, on_run)
    del xs, ys
    timed = times[warm:] if len(times) > warm else times
    sec = statistics.median(timed)
    value = BYTES_PER_ELEM * N_AXPY / sec / 1e9
    cb = {"value": round(value, 2), "unit": "GB/s", "cores": cpu_threads(), "kind": kind,
          "sample": f"full workload n=2^28 fp32, median of {len(timed)} enqueue+wait runs after {len(times) - len(timed)} "
                    f"warm-up (reference AxpyKernel functor (float) on the reference BlocksParallel engine, ept=4096)"}
    first_ok = checks.get(0) == [g[2] for g in gathered]
    final_ok = checks.get(applied - 1) == [g[3] for g in gathered]
    parity = {"check": (f"per-rank blake2b of GPU Y vs the reference CPU Y over the same index range, after the "
                        f"first step and after all {applied} steps (parity + warm-up + timed; Y compounds)"),
              "ranks": len(gathered), "first_step_match": bool(first_ok), "final_match": bool(final_ok),
              "match": bool(first_ok and final_ok)}
    return cb, parity


def cpu_baseline_dgemm(a, b, c, alpha, beta, Cb, q, task, bw_task=None):
    """Reference GemmTiledKernel (tile 32, BlocksParallel, all cores) on a 64-row sample of
    the 8192^3 workload; rows of the GPU result (from pristine C) checked against it."""
    from oracle import oracle as O
    rows = 64
    size = a.shape[0]
    # GPU result from pristine C for the parity rows
    Cb.upload(c)
    q.enqueue(task)
    q.wait()
    gpu_rows = Cb.download()[:rows]
    out = np.ascontiguousarray(c[:rows]).copy()
    sec = C.c_double()
    kind = "reference" if O.ref_available() else "port"
    if kind == "reference":
        r = O.ref()
        os.environ.setdefault("KERNELWEAVE_POOL_SIZE", str(cpu_threads()))
        assert r.kwref_gemm_kernel(1, 1, rows, size, size, alpha, beta, np.ascontiguousarray(a[:rows]).ctypes.data,
                                   size, b.ctypes.data, size, out.ctypes.data, size, 32, 16, 8, C.byref(sec)) == 0
        secs = sec.value
    else:
        t = time.perf_counter()
        out = O.gemm(alpha, beta, a[:rows], b, c[:rows], threads=cpu_threads())
        secs = time.perf_counter() - t
    tf = 2 * rows * size * size / secs / 1e12
    err = np.abs(gpu_rows - out)
    bound = (size + 4) * 2.0 ** -53 * np.abs(out)
    ok = bool(np.all(err <= bound))
    worst = float(np.max(err / bound))
    bitwise = None
    if bw_task is not None:
        Cb.upload(c)
        q.enqueue(bw_task)
        q.wait()
        bitwise = bool(np.array_equal(Cb.download()[:rows], out))
    cb = {"value": round(tf * 1e3, 3), "unit": "GFLOP/s", "cores": cpu_threads(), "kind": kind,
          "sample": f"{rows} of {size} rows of the 8192^3 workload (GemmTiledKernel tile 32, BlocksParallel); "
                    f"{secs:.2f} s"}
    return cb, {"check": "|dC| <= (K+4)*2^-53*|C_ref| on the sampled rows (DMMA kernel); bitwise equality "
                         "on the same rows (bit-exact mode)", "match": ok, "max_err_over_bound": round(worst, 4),
                "bitwise_mode_match": bitwise}


def run_reference(args, dist) -> dict | None:
    """The reference arm: the reference's own CPU AXPY (oracle/_ref, BlocksParallel on every host
    core) on the same global input, --warmup untimed + --steps timed enqueue+wait runs; rank 0
    only. `config`, `metric`, `unit` and `steps` are the product arm's."""
    if dist.rank != 0:
        return None
    xs, ys = axpy_inputs(0, N_AXPY)
    alpha = np.float32(9.096465)
    warm = max(1, args.warmup)
    times, kind = _ref_axpy_f32(xs, ys, alpha, warm + args.steps)
    del xs, ys
    sec = statistics.median(times[warm:])
    value = BYTES_PER_ELEM * N_AXPY / sec / 1e9
    cb = {"value": round(value, 2), "unit": "GB/s", "cores": cpu_threads(), "kind": kind,
          "sample": f"full workload n=2^28 fp32, median of {args.steps} runs after {warm} warm-up (reference "
                    f"BlocksParallel engine, AxpyKernel functor for float, ept=4096)"}
    dg = None
    try:
        from oracle import oracle as O
        if O.ref_available():
            size, rows = 8192, 64
            g = np.random.default_rng(77)
            a = g.random((rows, size)) * 10
            b = g.random((size, size)) * 10
            c = g.random((rows, size)) * 10
            gsec = C.c_double()
            assert O.ref().kwref_gemm_kernel(1, 1, rows, size, size, 1.25, 0.75, a.ctypes.data, size, b.ctypes.data,
                                             size, c.ctypes.data, size, 32, 16, 8, C.byref(gsec)) == 0
            dg = {"metric": "DGEMM fp64 TFLOP/s (2*M*N*K)", "value": round(2 * rows * size * size / gsec.value / 1e12, 5),
                  "unit": "TFLOP/s", "sample": f"{rows} rows of 8192^3, GemmTiledKernel tile 32, BlocksParallel, "
                                               f"{cpu_threads()} threads"}
    except Exception as ex:  # noqa: BLE001
        dg = {"error": str(ex)[:200]}
    return {"impl": "reference", "metric": "AXPY fp32 HBM GB/s (n=2^28, Y=alpha*X+Y, 12 B/elem)",
            "value": round(value, 2), "unit": "GB/s", "n_gpus": dist.world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(sec * 1e3, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": AXPY_DATA,
            "config": axpy_config(dist.world, args.tpb, args.ept),
            "cpu_baseline": cb, "e2e": {"value": round(value, 2), "unit": "GB/s", "h2d_bytes_per_step": 0,
                                        "d2h_bytes_per_step": 0}, "dgemm": dg}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--tpb", type=int, default=512)
    ap.add_argument("--ept", type=int, default=4)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--dgemm-steps", type=int, default=10)
    ap.add_argument("--panels", type=int, default=8)
    ap.add_argument("--dgemm-timeout", type=float, default=300.0,
                    help="seconds the DGEMM leg may take before the headline line is printed without it")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--no-dgemm", action="store_true")
    ap.add_argument("--no-f64", action="store_true")
    ap.add_argument("--no-cublas", action="store_true")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl")
    ap.add_argument("--same-gpu", action="store_true", help="self-test: all ranks on GPU 0 (gloo only)")
    ap.add_argument("--force-rowsharded", action="store_true",
                    help="self-test: run the 16384^3 row-sharded NCCL path even at world size 1")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        if rank != 0:
            return 0
        class _D:  # no process group needed: rank 0 alone runs the CPU reference
            world = int(os.environ.get("WORLD_SIZE", "1"))
            rank = 0
        out = run_reference(args, _D())
        print(json.dumps(out), flush=True)
        return 0
    if args.same_gpu and args.dist_backend != "gloo":
        ap.error("--same-gpu requires --dist-backend gloo")
    dist = Dist(args.gpus, args.dist_backend, args.same_gpu)
    try:
        out = run_ours(args, dist)
    finally:
        pass
    if dist.rank == 0:
        print(json.dumps(out), flush=True)
    dist.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
