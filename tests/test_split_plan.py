"""CPU: the SPLIT DGEMM schedule (kw_dgemm_split_plan — the same split_range the kernel runs).
Properties the kernel's correctness and deadlock-freedom rest on:
  * every (tile, k-tile) of the problem is computed by exactly one piece;
  * a tile is split at most once: a tail piece [x, K) of CTA c finishes the tile whose head
    piece [0, x) is CTA c - 1's — parked in slot c - 1, which is the slot the kernel reloads;
  * a head piece is its CTA's first stream-K piece and a tail its last, so the CTA a tail waits
    on has no wait before its head (no cycle, hence no deadlock with start-order tickets)."""
import ctypes as C

import numpy as np
import pytest

from paper_1602_08477_b200 import _lib as L


def plan(T, K, G, c, dp=-1):
    out = (C.c_int * 11)()
    assert L.lib().kw_dgemm_split_plan(T, K, G, c, dp, out) == 0
    return dict(zip(["ndp", "dp0", "dp_step", "head", "nfull", "tail", "t_head", "x_head", "t_full0", "t_tail",
                     "x_tail"], list(out)))


@pytest.mark.parametrize("T,K,G,dp", [(256, 64, 148, -1), (1024, 128, 148, -1), (512, 128, 296, -1),
                                      (16384, 512, 148, -1), (149, 3, 148, -1), (1000, 7, 444, -1),
                                      (16384, 512, 148, 0), (5000, 33, 148, 2960), (300, 2, 148, 10 ** 9)])
def test_split_plan_covers_each_k_tile_once(T, K, G, dp):
    cover = np.zeros((T, K), dtype=np.int32)
    plans = [plan(T, K, G, c, dp) for c in range(G)]
    for c, p in enumerate(plans):
        for j in range(p["ndp"]):
            cover[p["dp0"] + j * p["dp_step"], :] += 1
        if p["head"]:
            assert 0 < p["x_head"] < K
            cover[p["t_head"], :p["x_head"]] += 1
        for t in range(p["t_full0"], p["t_full0"] + p["nfull"]):
            cover[t, :] += 1
        if p["tail"]:
            assert 0 < p["x_tail"] < K and c > 0
            prev = plans[c - 1]
            assert prev["head"] == 1 and prev["t_head"] == p["t_tail"] and prev["x_head"] == p["x_tail"]
            cover[p["t_tail"], p["x_tail"]:] += 1
            assert p["t_tail"] != p["t_head"] or not p["head"]
    assert (cover == 1).all()
    # balance: stream-K ranges differ by at most one k-tile
    work = [p["ndp"] * K + (p["x_head"] if p["head"] else 0) + p["nfull"] * K + ((K - p["x_tail"]) if p["tail"] else 0)
            for p in plans]
    assert max(work) - min(work) <= 1


def test_split_plan_rejects_fewer_tiles_than_ctas():
    out = (C.c_int * 11)()
    assert L.lib().kw_dgemm_split_plan(100, 8, 148, 0, -1, out) == L.KW_USAGE
