"""Summarise an ncu --set full report into the numbers DESIGN.md / bench.py cite.
usage: python tools/ncu_summary.py report.ncu-rep [label] -> JSON on stdout."""
import csv
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct_of_peak",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum": "smem_ld_bank_conflicts",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum": "smem_ld_wavefronts",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "s": 1, "second": 1, "Ghz": 1e9, "Mhz": 1e6, "hz": 1}


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    res = {"report": rep.split("/")[-1], "kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else None}
    stalls = {}
    for name, unit, val in zip(hdr, units, vals):
        if name in KEYS:
            try:
                v = float(val.replace(",", "")) * SCALE.get(unit, 1)
            except ValueError:
                continue
            res[KEYS[name]] = v
        if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("not_issued"):
            try:
                stalls[name.replace("smsp__pcsamp_warps_issue_stalled_", "")] = int(val.replace(",", ""))
            except ValueError:
                pass
    tot = sum(stalls.values()) or 1
    res["stall_top"] = {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:6]}
    if "dram_read" in res and "dram_write" in res:
        res["dram_bytes_per_launch"] = res["dram_read"] + res["dram_write"]
    if len(sys.argv) > 2:
        res["label"] = sys.argv[2]
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
