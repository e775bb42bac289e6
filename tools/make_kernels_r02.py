"""profiles/r02_kernels.md + profiles/r02_traffic.json from the round-2 ncu captures
(profiles/r02_ncu_captures.json, written by tools/summarize_r02.py).

Each capture is one launch at steady-state history depth d; the algorithmic bytes / flops are DESIGN.md
section 3's per-launch model at that (n, m, d).  HBM fraction = algorithmic bytes / time / measured copy peak;
FP64 fraction = algorithmic flops / time / measured DMMA peak; the binding one is the larger model time.
"""
import json
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
HBM = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() \
    else 6541.5
FP64 = json.loads((ROOT / "profiles" / "fp64_peak.json").read_text())["dmma_tflops"]


def model(tag, n, m, d, nnz=0, mat=0):
    nm = float(n) * m
    return {
        "hist_update": (8.0 * (d + 2) * nm, 2.0 * d * m * nm),
        "hist_gram": (8.0 * (d + 1) * nm, 2.0 * d * m * nm),
        "tri_apply": (16.0 * nm, 1.0 * m * nm),
        "xr": (8.0 * (2 * nm + 4 * n), 4.0 * nm),
        "stencil": (16.0 * nm + mat, 2.0 * nnz * m),
        "csr": (16.0 * nm + mat, 2.0 * nnz * m),
    }[tag]


# capture file stem -> (config label, tag, n, m, d, nnz, matrix bytes)
N5, N5Q, N3, N4 = 8192 ** 2, 4096 ** 2, 128 ** 3, 256 ** 3
CASES = {
    "r02_cfg5full_hist_update": ("5 (8192^2, lean)", "hist_update", N5, 64, 3, 0, 0),
    "r02_cfg5full_stencil": ("5 (8192^2)", "stencil", N5, 64, 0, 5 * N5 - 4 * 8192, 512 * 512 * 8),
    "r02_cfg5full_stencil_waves": ("5 (8192^2), whole-wave chunks", "stencil", N5, 64, 0, 5 * N5 - 4 * 8192, 512 * 512 * 8),
    "r02_cfg5full_stencil_hoisted": ("5 (8192^2), + tile-layer hoisting", "stencil", N5, 64, 0, 5 * N5 - 4 * 8192, 512 * 512 * 8),
    "r02_cfg5full_hist_gram": ("5 (8192^2, lean)", "hist_gram", N5, 64, 3, 0, 0),
    "r02_cfg5full_tri_apply": ("5 (8192^2, lean)", "tri_apply", N5, 64, 0, 0, 0),
    "r02_cfg5_hist_gram": ("5 (4096^2)", "hist_gram", N5Q, 64, 3, 0, 0),
    "r02_cfg5_xr": ("5 (4096^2)", "xr", N5Q, 64, 0, 0, 0),
    "r02_cfg3_hist_update": ("3 (128^3)", "hist_update", N3, 32, 4, 0, 0),
    "r02_cfg3_hist_gram": ("3 (128^3)", "hist_gram", N3, 32, 4, 0, 0),
    "r02_cfg3_stencil": ("3 (128^3)", "stencil", N3, 32, 0, 7 * N3 - 6 * 128 ** 2, 8 * N3),
    "r02_cfg3_stencil_waves": ("3 (128^3), whole-wave chunks", "stencil", N3, 32, 0, 7 * N3 - 6 * 128 ** 2, 8 * N3),
    "r02_cfg3_stencil_hoisted": ("3 (128^3), + tile-layer hoisting", "stencil", N3, 32, 0, 7 * N3 - 6 * 128 ** 2, 8 * N3),
    "r02_cfg4_hist_update": ("4 (256^3)", "hist_update", N4, 64, 2, 0, 0),
    "r02_cfg4_hist_gram": ("4 (256^3)", "hist_gram", N4, 64, 2, 0, 0),
    "r02_cfg4_stencil": ("4 (256^3)", "stencil", N4, 64, 0, 7 * N4 - 6 * 256 ** 2, 0),
    "r02_csr_m64": ("5 (2048^2, CSR)", "csr", 2048 ** 2, 64, 0, 5 * 2048 ** 2 - 4 * 2048,
                    12 * (5 * 2048 ** 2 - 4 * 2048) + 8 * (2048 ** 2 + 1)),
}


def main():
    caps = json.loads((ROOT / "profiles" / "r02_ncu_captures.json").read_text())
    rows, traffic = [], {}
    for c in caps:
        stem = c["capture"].replace(".ncu-rep", "")
        if stem not in CASES:
            continue
        cfg, tag, n, m, d, nnz, mat = CASES[stem]
        b, f = model(tag, n, m, d, nnz, mat)
        t = c["time_ms"] / 1e3
        hbm_frac, fp_frac = b / t / 1e9 / HBM, f / t / 1e12 / FP64
        bound = "fp64" if f / (FP64 * 1e12) > b / (HBM * 1e9) else "hbm"
        dram = c["dram_gb"] * 1e9
        rows.append((cfg, tag, c["kernel"].replace("void <unnamed>::", "").replace("void ", ""), d, c["time_ms"],
                     b / 1e9, dram / 1e9, dram / b, hbm_frac, fp_frac, c.get("dmma_pipe_active", 0.0), bound))
        if stem in ("r02_cfg5full_hist_update", "r02_cfg5full_hist_gram", "r02_cfg5full_tri_apply"):
            traffic[f"cfg5-trunc3-srecg2-t64-tiled2d-8192, 8-iteration window from x0=0|{tag}"] = {
                "dram_bytes_per_launch": dram, "alg_bytes": b, "d": d, "time_ms": c["time_ms"],
                "source": f"profiles/{stem}.ncu-rep (ncu --set full --clock-control none, one launch at d = {d})"}
    lines = ["# Round-2 ncu captures: one launch per hot kernel at steady-state depth d", "",
             f"Peaks: HBM {HBM} GB/s (MEASURED_PEAKS.json), FP64 DMMA {FP64} TFLOP/s (profiles/fp64_peak.json). "
             "Algorithmic bytes / flops per launch are DESIGN.md section 3's model; 'frac' columns divide them by "
             "the captured duration (ncu serialises launches and runs cold-cache, so these are per-launch rates, "
             "not the in-solve shares -- see r02_launches_cfg5.md).", "",
             "| config | kernel (tag) | template | d | time ms | alg GB | DRAM GB | DRAM / alg | HBM frac | "
             "FP64 frac | DMMA pipe | bound |", "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        lines.append(f"| {r[0]} | {r[1]} | `{r[2][:60]}` | {r[3]} | {r[4]:.3f} | {r[5]:.2f} | {r[6]:.2f} | "
                     f"{r[7]:.3f} | {r[8]:.2f} | {r[9]:.2f} | {r[10]:.2f} | {r[11]} |")
    (ROOT / "profiles" / "r02_kernels.md").write_text("\n".join(lines) + "\n")
    if traffic:
        (ROOT / "profiles" / "r02_traffic.json").write_text(json.dumps(traffic, indent=1))
    print("\n".join(lines))


if __name__ == "__main__":
    main()
