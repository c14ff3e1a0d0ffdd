"""Per-instruction stall samples of each kernel in an ncu report (sass source page).

    python tools/ncu_source.py report.ncu-rep [kernel-substring] [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
pat = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
blocks = raw.split('"Kernel Name",')
for b in blocks[1:]:
    name = b.split("\n", 1)[0]
    if pat not in name:
        continue
    rows = list(csv.reader(io.StringIO(b.split("\n", 1)[1])))
    hdr = rows[0]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ie = hdr.index("Instructions Executed")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(float(r[si] or 0) for r in rows[1:] if len(r) > si)
    agg = {}
    for r in rows[1:]:
        for i in stall_cols:
            agg[hdr[i]] = agg.get(hdr[i], 0) + float(r[i] or 0)
    print("=====", name[:90], "samples", tot)
    print("  stall mix:", ", ".join(f"{k[6:]} {100 * v / tot:.1f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
    hot = sorted(rows[1:], key=lambda r: -float(r[si] or 0))[:top]
    for r in hot:
        st = sorted(((hdr[i][6:], float(r[i] or 0)) for i in stall_cols), key=lambda kv: -kv[1])[:3]
        print(f"  {float(r[si]):7.0f} {r[1].strip()[:60]:60s} exec={r[ie]:>9s} " + " ".join(f"{k}:{v:.0f}" for k, v in st if v))
