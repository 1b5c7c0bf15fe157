"""Multi-GPU decomposition of the hot path (one process per GPU).

AXPY: contiguous index ranges, boundaries on 16-byte multiples; no collective — every element
is independent, so the sharded result is bit-identical to one GPU by construction.

DGEMM: rank r owns row block r of A and C (boundaries on the 128-row tile); B lives on the root
and is broadcast (ncclBroadcast over NVLink). Default "kslab" schedule: two row slabs of B
(dgemm_kslabs — contiguous rows, broadcast in place from the root's B), the rank's product run as
two k-range launches. KW_ROWSHARD_SCHEDULE=panels: column panels, panel j stored k x w_j at leading
dimension round8(w_j) in the panel-major scratch (the Buffer pitch rule, so an odd-width last
panel stays TMA-addressable), each panel's broadcast overlapped with the previous panel's DGEMM.
`dgemm_panels` is the exact layout kw_dgemm_rowsharded uses (kw_comm.cu), so host code and
tests can reproduce it.
"""
from __future__ import annotations

import os
from dataclasses import dataclass


def ceil_div(a: int, b: int) -> int:
    return -(-a // b)


def axpy_range(n: int, world: int, rank: int, align: int = 4) -> tuple[int, int]:
    """[lo, hi) of `rank`; shard sizes are multiples of `align` elements except the last."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank must lie in [0, world)")
    per = ceil_div(ceil_div(n, world), align) * align
    lo = min(n, rank * per)
    return lo, min(n, lo + per)


def dgemm_rows(m: int, world: int, rank: int, tile: int = 128) -> tuple[int, int]:
    """Row block [r0, r1) of A and C owned by `rank` (tile-aligned boundaries)."""
    return axpy_range(m, world, rank, align=tile)


@dataclass(frozen=True)
class Panel:
    index: int
    n0: int          # first column of B / C
    width: int       # columns in this panel
    offset: int      # element offset of the k x width panel in the panel-major scratch
    ld: int = 0      # its leading dimension: width rounded up to 8 doubles (Buffer pitch rule)


def dgemm_panels(n: int, k: int, panels: int, tile: int = 128) -> list[Panel]:
    """Column panels of B exactly as kw_dgemm_rowsharded lays them out (kw_comm.cu panel_bounds):
    equal tile-aligned widths of ceil(n / panels), each at leading dimension round8(width)."""
    if panels < 1:
        raise ValueError("panels must be >= 1")
    w = ceil_div(ceil_div(n, panels), tile) * tile
    out, off = [], 0
    for j, n0 in enumerate(range(0, n, w)):
        wj = min(w, n - n0)
        ld = ceil_div(wj, 8) * 8
        out.append(Panel(j, n0, wj, off, ld))
        off += k * ld
    return out


def dgemm_kslabs(k: int, panels: int) -> list[tuple[int, int]]:
    """Row slabs [k0, k1) of B the default "kslab" schedule broadcasts (kw_comm.cu
    first_slab_ktiles): the first 1/panels of the 16-row k-tiles, then the rest."""
    ktiles = ceil_div(k, 16)
    if panels <= 1 or ktiles < 2:
        return [(0, k)]
    a = max(1, ktiles // panels) * 16
    return [(0, min(a, k))] + ([(a, k)] if a < k else [])


def kslab_schedule() -> bool:
    return os.environ.get("KW_ROWSHARD_SCHEDULE") != "panels"


def dgemm_panel_scratch(n: int, k: int, panels: int, tile: int = 128) -> int:
    """Doubles of B scratch kw_dgemm_rowsharded needs (kw_dgemm_rowsharded_scratch): B at the
    Buffer pitch (k x round8(n)) for the default k-slab schedule, the panel-major layout for
    KW_ROWSHARD_SCHEDULE=panels."""
    if n == 0:
        return 0
    if kslab_schedule():
        return k * ceil_div(n, 8) * 8
    return sum(k * p.ld for p in dgemm_panels(n, k, panels, tile))
