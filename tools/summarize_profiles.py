"""Summarise ncu outputs from gpurun_out/ into tracked files under profiles/.

    python tools/summarize_profiles.py <tag> [launches.csv] [prof.ncu-rep]

Writes profiles/<tag>_launches.md (per-kernel share of the step, from the
`--metrics gpu__time_duration.sum` launch list) and profiles/<tag>_ncu.md +
profiles/ncu_summary.json (per-kernel DRAM traffic, pipe utilisation and
stall mix from one `--set full` capture). bench.py reads the traffic figure
for its roofline object from profiles/ncu_summary.json.
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
PROF = ROOT / "profiles"

METRICS = {
    "time_ms": ("gpu__time_duration.sum", 1e-6),
    "dram_read_B": ("dram__bytes_read.sum", 1.0),
    "dram_write_B": ("dram__bytes_write.sum", 1.0),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
    "alu_pct": ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "fma_pct": ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "fmaheavy_pct": ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", 1.0),
    "fp64_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "regs": ("launch__registers_per_thread", 1.0),
    "grid": ("launch__grid_size", 1.0),
    "inst": ("smsp__inst_executed.sum", 1.0),
    "sm_ghz": ("sm__cycles_elapsed.avg.per_second", 1.0),
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "usecond": 1e3, "msecond": 1e6,
              "Ghz": 1, "Mhz": 1e-3, "hz": 1e-9}


def launches(path: Path) -> str:
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    t, c = defaultdict(float), defaultdict(int)
    for r in rows[start + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            t[r[ki]] += float(r[vi].replace(",", ""))
            c[r[ki]] += 1
    tot = sum(t.values())
    out = ["| kernel | launches | total ms | mean us/launch | share |", "|---|---:|---:|---:|---:|"]
    for k in sorted(t, key=t.get, reverse=True):
        out.append(f"| `{k}` | {c[k]} | {t[k] / 1e6:.3f} | {t[k] / c[k] / 1e3:.1f} | {100 * t[k] / tot:.1f}% |")
    return "\n".join(out)


def full(path: Path) -> list[dict]:
    raw = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for key, (m, _) in METRICS.items():
            if m not in hdr:
                continue
            i = hdr.index(m)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            u = units[i]
            if key.endswith("_B"):
                v *= UNIT_SCALE.get(u, 1)
            if key == "time_ms":
                v = v * {"ns": 1e-6, "nsecond": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(u, 1e-6)
            d[key] = v
        stalls = {h.split("smsp__average_warps_issue_stalled_")[1].split("_per_issue_active")[0]: float(r[hdr.index(h)])
                  for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("per_issue_active.ratio")
                  and r[hdr.index(h)] not in ("", "n/a")}
        d["top_stalls"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:4])
        res.append(d)
    return res


def main() -> None:
    tag = sys.argv[1]
    lcsv = Path(sys.argv[2]) if len(sys.argv) > 2 else ROOT / "gpurun_out" / "launches.csv"
    rep = Path(sys.argv[3]) if len(sys.argv) > 3 else ROOT / "gpurun_out" / "prof_full.ncu-rep"
    PROF.mkdir(exist_ok=True)
    if lcsv.exists():
        (PROF / f"{tag}_launches.md").write_text(
            f"# {tag}: kernel launch list (ncu --metrics gpu__time_duration.sum --clock-control none)\n\n"
            f"Command: `ncu ... python bench.py --quick --steps 2 --warmup 1` (cold-cache, serialised; compare shares).\n\n"
            + launches(lcsv) + "\n")
    if rep.exists():
        ks = full(rep)
        lines = [f"# {tag}: ncu --set full summary (tools/prof_kernels.py, one launch per kernel)\n",
                 "| kernel | ms | DRAM write GB | DRAM read MB | issue % | ALU % | FMA % | FMA-heavy % | FP64 % | warps % | regs | top stalls |",
                 "|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|---|"]
        for d in ks:
            lines.append(
                f"| `{d['kernel'][:60]}` | {d.get('time_ms', 0):.3f} | {d.get('dram_write_B', 0) / 1e9:.3f} | "
                f"{d.get('dram_read_B', 0) / 1e6:.1f} | {d.get('issue_active_pct', 0):.1f} | {d.get('alu_pct', 0):.1f} | "
                f"{d.get('fma_pct', 0):.1f} | {d.get('fmaheavy_pct', 0):.1f} | {d.get('fp64_pct', 0):.1f} | "
                f"{d.get('warps_active_pct', 0):.1f} | {d.get('regs', 0):.0f} | "
                + ", ".join(f"{k} {v:.1f}" for k, v in d["top_stalls"].items()) + " |")
        (PROF / f"{tag}_ncu.md").write_text("\n".join(lines) + "\n")
        names = {"fill_kernel<0, 1": "uniform_f32_philox", "fill_kernel<1, 1": "uniform_f32_threefry",
                 "fill_kernel<2, 1": "uniform_f32_squares", "staged_prefix_kernel<3, 1": "uniform_f32_tyche",
                 "tyche_prefix_kernel<1": "uniform_f32_tyche"}
        traffic = {}
        for d in ks:
            for pat, nm in names.items():
                if pat in d["kernel"] and nm not in traffic:
                    traffic[nm] = d.get("dram_read_B", 0) + d.get("dram_write_B", 0)
        (PROF / "ncu_summary.json").write_text(json.dumps({"tag": tag, "traffic_bytes": traffic, "kernels": ks},
                                                          indent=1) + "\n")
    print("wrote profiles for", tag)


if __name__ == "__main__":
    main()
