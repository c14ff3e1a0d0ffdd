"""Per-word pipe work of the headline fill kernels, from their SASS main loops.

    python tools/sass_pipes.py

Counts, per output word, the ALU-pipe instructions (LOP3/SHF/IADD3/LEA/ISETP/...),
the FMA-heavy slots (IMAD 1, IMAD.HI 2, IMAD.WIDE 2.5: the measured rates of
profiles/r1s_probe_pipes.json), FP64 and XU instructions and the total issued, in
the main loop of each default kernel instantiation (the hottest backward-branch
body, or an explicit address range). bench.py's INT_WORK_PER_WORD holds the output.
"""
from __future__ import annotations

import re
import subprocess
from collections import Counter
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
FILL = ROOT / "paper_2310_19925_b200/_lib/obj/cbrng_fill.o"
MULTI = ROOT / "paper_2310_19925_b200/_lib/obj/cbrng_multistream.o"
ALU = ("LOP3", "SHF", "IADD3", "I2FP", "PRMT", "LEA", "ISETP", "SEL", "FSEL", "VIMNMX", "IMNMX", "FMNMX",
       "BMSK", "SGXT", "FLO", "POPC")


def mix(obj: Path, fun: str, lo: int | None = None, hi: int | None = None) -> Counter:
    out = subprocess.run(["cuobjdump", "-sass", "-fun", fun, str(obj)], capture_output=True, text=True).stdout
    ins = []
    for line in out.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)(.*)", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(3), m.group(4)))
    if lo is None:  # largest loop body
        best = None
        for a, op, rest in ins:
            t = re.search(r"0x([0-9a-f]+)", rest) if op.startswith("BRA") else None
            if t and int(t.group(1), 16) < a and (best is None or a - int(t.group(1), 16) > best[1] - best[0]):
                best = (int(t.group(1), 16), a)
        lo, hi = best
    return Counter(op for a, op, _ in ins if lo <= a <= hi)


def pipes(c: Counter, per: float) -> dict:
    def slots(k):
        return 2.5 if k.startswith("IMAD.WIDE") else 2.0 if k.startswith("IMAD.HI") else 1.0

    return {
        "alu": round(sum(v for k, v in c.items() if k.split(".")[0] in ALU) / per, 2),
        "fma_heavy_slots": round(sum(v * slots(k) for k, v in c.items() if k.startswith(("IMAD", "VIADD"))) / per, 2),
        "fp64": round(sum(v for k, v in c.items() if k.split(".")[0] in ("DFMA", "DMUL", "DADD")) / per, 2),
        "xu": round(sum(v for k, v in c.items() if (k.startswith("I2F") and not k.startswith("I2FP"))
                        or k.startswith("MUFU")) / per, 2),
        "issue": round(sum(c.values()) / per, 2),
    }


def main() -> None:
    # default instantiations (cbrng_fill.cu / cbrng_multistream.cu defaults)
    print("philox  ", pipes(mix(FILL, "_ZN5cbrng11fill_kernelILi0ELi1ELi16ELb0ELi0ELi4ELi0EEEvNS_8FillArgsIXT_EEE"), 64))
    print("threefry", pipes(mix(FILL, "_ZN5cbrng11fill_kernelILi1ELi1ELi12ELb0ELi4ELi4ELi0EEEvNS_8FillArgsIXT_EEE"), 48))
    print("squares ", pipes(mix(FILL, "_ZN5cbrng11fill_kernelILi2ELi1ELi16ELb0ELi2ELi4ELi0EEEvNS_8FillArgsIXT_EEE"), 64))
    ty = "_ZN5cbrng20staged_prefix_kernelILi3ELi1ELb1ELi1ELi4ELi256EEEvNS_10PrefixArgsE"
    # Tyche (256-word rows, CV 1): the full-warp 16-word staging loop, plus the
    # per-row warm-up (tyche_init: a 4-mix loop body run 5 times) spread over the
    # row. Addresses of the build this was read from (r1w); re-read them from
    # `cuobjdump -sass` after changes.
    print("tyche group ", pipes(mix(MULTI, ty, 0x35F0, 0x4660), 16))
    print("tyche warmup", pipes(mix(MULTI, ty, 0x440, 0x760), 256 / 5))


if __name__ == "__main__":
    main()
