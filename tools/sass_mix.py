"""Opcode histogram of one kernel's SASS (between two labels if given).

    python tools/sass_mix.py <object or .so> <function-substring>
"""
import re
import subprocess
import sys
from collections import Counter

obj, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if pat not in name:
        continue
    ops = Counter()
    for line in f.splitlines():
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
        if m:
            ops[m.group(2)] += 1
    print(name, sum(ops.values()))
    for k, v in ops.most_common():
        print(f"  {v:5d} {k}")
