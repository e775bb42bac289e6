"""Summarise round-2 ncu --set full captures (one launch each) into a JSON / markdown table.

    python tools/summarize_r02.py gpurun_out/r02_*.ncu-rep
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

KEYS = {
    "time_ms": "gpu__time_duration.sum",
    "dram_read_gb": "dram__bytes_read.sum",
    "dram_write_gb": "dram__bytes_write.sum",
    "dmma_active_cycles": "SM_C.TriageCompute.smsp__pipe_tensor_subpipe_dmma_cycles_active.avg",
    "elapsed_cycles": "sm__cycles_elapsed.avg",
    "sm_ghz": "sm__cycles_elapsed.avg.per_second",
    "fp64_tensor_ops": "sm__ops_path_tensor_src_fp64.sum",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "occupancy_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "long_scoreboard": "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "math_throttle": "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "barrier": "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "wait": "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "short_scoreboard": "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "inst_executed": "smsp__inst_executed.sum",
}
SCALE = {"Gbyte": 1.0, "Mbyte": 1e-3, "Kbyte": 1e-6, "byte": 1e-9, "ms": 1.0, "us": 1e-3, "usecond": 1e-3,
         "msecond": 1.0, "nsecond": 1e-6, "ns": 1e-6}


def one(path):
    out = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    col = {h: i for i, h in enumerate(hdr)}
    d = {"capture": Path(path).name, "kernel": vals[col["Kernel Name"]].split("(")[0]}
    for k, h in KEYS.items():
        if h not in col:
            continue
        v, u = vals[col[h]].replace(",", ""), units[col[h]]
        try:
            x = float(v)
        except ValueError:
            continue
        if k.endswith("_gb") or k == "time_ms":
            x *= SCALE.get(u, 1.0)
        d[k] = x
    if "dmma_active_cycles" in d and "elapsed_cycles" in d:
        d["dmma_pipe_active"] = d["dmma_active_cycles"] / d["elapsed_cycles"]
    d["dram_gb"] = d.get("dram_read_gb", 0) + d.get("dram_write_gb", 0)
    d["dram_tbs"] = d["dram_gb"] / d["time_ms"]
    if d.get("fp64_tensor_ops"):
        d["dmma_tflops"] = d["fp64_tensor_ops"] / d["time_ms"] / 1e9
    return d


if __name__ == "__main__":
    res = [one(p) for p in sys.argv[1:]]
    print(json.dumps(res, indent=1))
