"""profiles/r01_traffic.json from the d = 100 full captures (tools/gpu_profile.sh):
DRAM bytes per launch of the two CGS2 kernels and their algorithmic bytes."""
import csv
import json
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
N, M, D = 64 ** 3, 16, 100


def dram_bytes(rep):
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(k)
        tot += float(vals[i]) * scale[units[i]]
    return int(tot), vals[hdr.index("Kernel Name")].split("(")[0]


out, names = {}, []
for tag, rep, nblk in (("hist_gram", "prof_hist_gram", D + 1), ("hist_update", "prof_hist_update", D + 2)):
    p = ROOT / "gpurun_out" / f"{rep}.ncu-rep"
    out[tag], name = dram_bytes(p)
    names.append(name.replace("void ", "").replace("<unnamed>::", ""))
    out[tag + "_alg"] = 8 * N * M * nblk
    out[tag + "_d"] = D
out["source"] = (f"ncu --set full --clock-control none, {names[0]} / {names[1]} at d={D} "
                 "(profiles/r01_prof_hist_*.ncu-rep)")
(ROOT / "profiles" / "r01_traffic.json").write_text(json.dumps(out) + "\n")
print(out)
