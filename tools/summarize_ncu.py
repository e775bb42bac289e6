"""Summarise ncu outputs into profiles/: kernel shares from a launch list and
key metrics of full captures.  Usage: python tools/summarize_ncu.py <round-tag>"""
import collections
import csv
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
out = ROOT / "profiles"
go = ROOT / "gpurun_out"


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hdr, seq = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                v = float(d["Metric Value"])
                unit = d["Metric Unit"]
                us = {"nsecond": v / 1e3, "ns": v / 1e3, "usecond": v, "us": v, "msecond": v * 1e3,
                      "ms": v * 1e3}.get(unit, v / 1e3)
                name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
                seq.append((name, d["Grid Size"], us))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for name, grid, us in seq:
        agg[name][0] += 1
        agg[name][1] += us
    tot = sum(v[1] for v in agg.values())
    lines = [f"# kernel shares of one config-2 solve (ncu launch list, cold-cache serialised; {len(seq)} launches, "
             f"{tot / 1e3:.1f} ms total)", "", "| kernel | launches | total ms | share | avg us |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {v[0]} | {v[1] / 1e3:.2f} | {100 * v[1] / tot:.1f} % | {v[1] / v[0]:.1f} |")
    return "\n".join(lines) + "\n"


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "lts__t_sector_hit_rate.pct", "launch__grid_size", "launch__block_size"]


def full_capture(path):
    txt = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:90], "grid": r[hdr.index("Grid Size")]}
        for w in WANT:
            if w in hdr:
                d[w] = f"{r[hdr.index(w)]} {units[hdr.index(w)]}".strip()
        res.append(d)
    return res


if __name__ == "__main__":
    md = launch_shares(go / f"launches_{tag}.csv")
    caps = {}
    for name in ("prof_hist_gram", "prof_hist_update"):
        p = go / f"{name}.ncu-rep"
        if p.exists():
            caps[name] = full_capture(p)
    md += "\n# full captures (ncu --set full)\n"
    for name, lst in caps.items():
        md += f"\n## {name}\n\n"
        for d in lst:
            md += "- " + "; ".join(f"{k}={v}" for k, v in d.items()) + "\n"
    (out / f"{tag}_ncu_summary.md").write_text(md)
    json.dump(caps, open(out / f"{tag}_ncu_captures.json", "w"), indent=1)
    print(md)
