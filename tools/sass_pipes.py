"""Per-unit pipe work of the hot kernels, read live from the built library's SASS.

    python tools/sass_pipes.py [path/to/libcbrng_b200.so]

bench.py imports this module and derives each kernel's per-unit pipe work from
the .so it actually loaded (cuobjdump -sass), so the compute-roofline fractions
it reports follow every kernel edit instead of a hard-coded table.

For a kernel, the hot loop is the innermost loop (a backward branch whose body
holds no other loop) with the most instructions; its opcode histogram divided
by the units one iteration produces gives the per-unit work per pipe:

  * alu       ALU-pipe instructions (LOP3, SHF, IADD3, I2FP, PRMT, LEA, ISETP, ...)
  * fma_heavy FMA-heavy-pipe slots: IMAD / IMAD.SHL / VIADD count 1, IMAD.HI 2,
              IMAD.WIDE 2 (RZ addend: a plain 32x32->64 product) or 2.5 (64-bit
              register addend) — the measured issue rates of these forms against
              IMAD's (profiles/r1s_probe_pipes.json, r1zd_probe_pipes.json); ncu's
              FMA-heavy utilisation of the Philox fill (79 %, r1zd) agrees with 2
  * fp64      DFMA / DMUL / DADD
  * xu        I2F (legacy conversions) and MUFU, each weighted by its measured
              rate (14.1 / 30.7 / 16 per clock per SM) into 63.3-op equivalents
  * issue     every instruction (the SM issues one warp-instruction per clock
              per sub-partition: 128 thread-instructions per clock per SM)

Units per hot-loop iteration come from the kernel's template arguments (the
demangled name): fill_kernel<ALG, OUT, ILP, ...> produces ILP 4-word units per
thread per iteration (ILP Box-Muller pairs when OUT = 3); the 256-word-row
staged_prefix_kernel 16 words per thread per group iteration; the fused
Brownian kernel 2 particle-steps (its step loop is `#pragma unroll 2`).
Tyche rows add the per-row warm-up (tyche_init's 20 mixes, a loop of
`mixes_per_body` mixes, counted from its SHF.L.W rotations) spread over the
row's 256 words.
"""

from __future__ import annotations

import functools
import re
import subprocess
import sys
from collections import Counter
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
DEFAULT_SO = ROOT / "paper_2310_19925_b200" / "_lib" / "libcbrng_b200.so"

ALU = ("LOP3", "SHF", "IADD3", "I2FP", "PRMT", "LEA", "ISETP", "SEL", "FSEL", "VIMNMX", "IMNMX", "FMNMX",
       "BMSK", "SGXT", "FLO", "POPC", "IABS", "LOP")
FP64 = ("DFMA", "DMUL", "DADD")

# Measured per-SM thread-op rates (profiles/r1s_probe_pipes.json / r1zd_probe_pipes.json):
# LOP3/SHF 63.3, IMAD 63.2, DFMA/DMUL 63.1-63.2, I2F.F64.U64 14.1, I2F.RM 30.7 per clock.
PIPE_RATE = {"alu": 63.3, "fma_heavy": 63.2, "fp64": 63.1, "xu": 63.3, "issue": 128.0}


@functools.lru_cache(maxsize=None)
def _sass(so: str) -> str:
    return subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True, check=True).stdout


@functools.lru_cache(maxsize=None)
def functions(so: str) -> dict:
    """demangled name -> list of (addr, opcode, operands)."""
    text = _sass(so)
    parts = re.split(r"\n\s+Function : (\S+)\n", text)
    mangled = parts[1::2]
    bodies = parts[2::2]
    dem = subprocess.run(["c++filt"], input="\n".join(mangled), capture_output=True, text=True).stdout.splitlines()
    out = {}
    for name, body in zip(dem, bodies):
        ins = []
        for line in body.splitlines():
            m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)(.*)", line)
            if m:
                ins.append((int(m.group(1), 16), m.group(3), m.group(4).split(";")[0].strip()))
        out[name] = ins
    return out


def find(so: str, pattern: str) -> tuple[str, list]:
    """The one kernel whose demangled name matches `pattern` (regex)."""
    hits = [k for k in functions(so) if re.search(pattern, k)]
    if len(hits) != 1:
        raise LookupError(f"{pattern!r}: {len(hits)} kernels match: {hits[:4]}")
    return hits[0], functions(so)[hits[0]]


def loops(ins: list) -> list[tuple[int, int]]:
    """(first, last) address of every loop closed by a backward branch."""
    out = []
    for a, op, rest in ins:
        if op.startswith("BRA"):
            t = re.search(r"0x([0-9a-f]+)", rest)
            if t and int(t.group(1), 16) < a:
                out.append((int(t.group(1), 16), a))
    return out


def innermost(ls: list) -> list[tuple[int, int]]:
    return [l for l in ls if not any(o != l and l[0] <= o[0] and o[1] <= l[1] for o in ls)]


def _form(op: str, operands: str) -> str:
    """IMAD.WIDE with a 64-bit register addend issues at 25.2 thread-ops/clk/SM, with
    RZ (a plain 32x32->64 product, Philox's mulhilo) at 31.6: tag the two forms."""
    if op.startswith("IMAD.WIDE"):
        return op + (".RZ" if operands.split(",")[-1].strip() == "RZ" else ".ADD64")
    return op


def mix(ins: list, lo: int, hi: int) -> Counter:
    return Counter(_form(op, rest) for a, op, rest in ins if lo <= a <= hi)


def hot_loop(ins: list, must=None) -> tuple[int, int]:
    """The largest innermost loop (optionally one containing an opcode prefix)."""
    cands = innermost(loops(ins))
    if must:
        cands = [l for l in cands if any(op.startswith(must) for a, op, _ in ins if l[0] <= a <= l[1])]
    if not cands:
        raise LookupError("no loop")
    return max(cands, key=lambda l: sum(1 for a, _, _ in ins if l[0] <= a <= l[1]))


def _xu_rate(k: str) -> float:
    """Measured XU thread-op rates per SM per clock: 64-bit conversions 14.1, 32-bit
    conversions 30.7 (profiles/r1zd_probe_pipes.json); MUFU 16 (quarter rate, assumed)."""
    if k.startswith("MUFU"):
        return 16.0
    return 14.1 if (".F64" in k or ".U64" in k or ".S64" in k) else 30.7


def pipes(c: Counter, per: float) -> dict:
    """Per-unit work: thread-ops per pipe (FMA-heavy in IMAD slots, XU in 63.3-op
    equivalents of its measured rates) and total issued instructions."""
    def slots(k):
        if k.startswith("IMAD.WIDE"):
            return 2.0 if k.endswith(".RZ") else 2.5
        return 2.0 if k.startswith("IMAD.HI") else 1.0

    xu = [(k, v) for k, v in c.items() if (k.startswith("I2F") and not k.startswith("I2FP")) or k.startswith("MUFU")]
    return {
        "alu": sum(v for k, v in c.items() if k.split(".")[0] in ALU) / per,
        "fma_heavy": sum(v * slots(k) for k, v in c.items() if k.startswith(("IMAD", "VIADD"))) / per,
        "fp64": sum(v for k, v in c.items() if k.split(".")[0] in FP64) / per,
        "xu": sum(v * PIPE_RATE["xu"] / _xu_rate(k) for k, v in xu) / per,
        "issue": sum(c.values()) / per,
    }


def _add(a: dict, b: dict, w: float) -> dict:
    return {k: a[k] + w * b[k] for k in a}


def fill_work(so: str, alg: int, out: int) -> dict:
    """Per word (OUT 0/1/2 words: 4 per unit) or per pair (OUT 3) of the block-aligned fill."""
    # Squares: the non-wrapping finite-difference variant (V 2) is the bulk path;
    # Box-Muller (OUT 3): normal_fill_kernel<ALG, ILP, SKIP, V, LC, SC, NT, MB, PIPE, CV>
    v = "2" if alg == 2 else r"\d+"
    if out == 3:
        name, ins = find(so, rf"normal_fill_kernel<{alg}, (\d+), false, {v}, \d+, \d+, \d+, \d+, false, 0>")
        ilp = int(re.search(rf"normal_fill_kernel<{alg}, (\d+),", name).group(1))
    else:
        name, ins = find(so, rf"fill_kernel<{alg}, {out}, (\d+), false, {v},")
        ilp = int(re.search(rf"fill_kernel<{alg}, {out}, (\d+),", name).group(1))
    lo, hi = hot_loop(ins)
    per = ilp if out == 3 else 4 * ilp
    return {"kernel": name, "unit": "pair" if out == 3 else "word", "loop": [hex(lo), hex(hi)],
            **{k: round(v, 3) for k, v in pipes(mix(ins, lo, hi), per).items()}}


def rows_work(so: str, alg: int, out: int) -> dict:
    """Per word of 256-word rows. Philox / Threefry: rowsplit_kernel<ALG, OUT, CV, LPR, MB>,
    whose row loop holds the row's stream setup and its 64 / LPR blocks per lane. The
    others: staged_prefix_kernel<..., 256>, the group loop (16 words per thread) plus,
    for Tyche, the per-row warm-up over 256 words."""
    if alg in (0, 1):
        name, ins = find(so, rf"rowsplit_kernel<{alg}, {out}, \d+, \d+, 0>")
        lpr = int(re.search(rf"rowsplit_kernel<{alg}, {out}, \d+, (\d+),", name).group(1))
        lo, hi = hot_loop(ins, must="STG")
        w = pipes(mix(ins, lo, hi), 4 * (64 // lpr))
        return {"kernel": name, "unit": "word", "loop": [hex(lo), hex(hi)], **{k: round(v, 3) for k, v in w.items()}}
    name, ins = find(so, rf"staged_prefix_kernel<{alg}, {out}, true, \d+, 4, 256>")
    # the kernel has two group loops: the generic one (per-row store predicates: an
    # ISETP per row slot) and the full-warp 256-word-row path that every launch of
    # 2^k x 32 rows takes (one ISETP, the loop test); time goes to the second
    cands = [l for l in innermost(loops(ins))
             if any(op.startswith("STG") for a, op, _ in ins if l[0] <= a <= l[1])
             and any(op.startswith("STS") for a, op, _ in ins if l[0] <= a <= l[1])]
    if not cands:
        raise LookupError("no staged group loop")
    lo, hi = min(cands, key=lambda l: (sum(1 for a, op, _ in ins if l[0] <= a <= l[1] and op.startswith("ISETP")),
                                       -(l[1] - l[0])))
    w = pipes(mix(ins, lo, hi), 16)
    res = {"kernel": name, "unit": "word", "loop": [hex(lo), hex(hi)]}
    if alg == 3:
        warm = [l for l in innermost(loops(ins)) if l != (lo, hi)
                and not any(op.startswith("STG") for a, op, _ in ins if l[0] <= a <= l[1])
                and any(op.startswith("SHF.L.W") for a, op, _ in ins if l[0] <= a <= l[1])]
        if warm:
            wl = max(warm, key=lambda l: l[1] - l[0])
            c = mix(ins, *wl)
            mixes = max(1, sum(v for k, v in c.items() if k.startswith("SHF.L.W")) // 4)
            w = _add(w, pipes(c, 1), (20 / mixes) / 256)
            res["warmup_loop"] = [hex(wl[0]), hex(wl[1])]
    return {**res, **{k: round(v, 3) for k, v in w.items()}}


def brownian_fused_work(so: str) -> dict:
    """Per particle-step of the fused Philox walk (step loop unrolled by 2)."""
    name, ins = find(so, r"brownian_fused_philox_kernel<true,")
    lo, hi = hot_loop(ins, must="DMUL")
    return {"kernel": name, "unit": "particle-step", "loop": [hex(lo), hex(hi)],
            **{k: round(v, 3) for k, v in pipes(mix(ins, lo, hi), 2).items()}}


def fractions(work: dict, units_per_s: float, sms: int, mhz: float) -> dict:
    """Utilisation of each pipe at `units_per_s` (per GPU): work x rate / (pipe rate x SMs x clock)."""
    clk = sms * mhz * 1e6
    return {p: round(work[p] * units_per_s / (PIPE_RATE[p] * clk), 3) for p in PIPE_RATE if p in work}


def main() -> None:
    so = sys.argv[1] if len(sys.argv) > 1 else str(DEFAULT_SO)
    for alg, nm in enumerate(("philox", "threefry", "squares")):
        print(nm, "f32", fill_work(so, alg, 1))
    print("philox normal2", fill_work(so, 0, 3))
    print("tyche rows f32", rows_work(so, 3, 1))
    print("philox rows u32", rows_work(so, 0, 0))
    print("brownian fused", brownian_fused_work(so))


if __name__ == "__main__":
    main()
