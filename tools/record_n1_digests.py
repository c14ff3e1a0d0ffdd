"""Record the N = 1 GPU digests of the strong-scaled side rows from a bench line.

    python tools/record_n1_digests.py gpurun_out/bench.json

configs[2] (Brownian stats) and configs[3] (Box-Muller normals) have no
full-size CPU digest (the oracle would need ~10^4 s for configs[2]); their
GPU-count invariance is checked against the N = 1 run of the same kernels,
recorded here into tests/golden/gpu_n1_digests.json. configs[4]'s reference
is the reference package's own full-size digest (golden_r2.json).
"""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
line = json.loads(Path(sys.argv[1]).read_text().strip().splitlines()[-1])
assert line["n_gpus"] == 1, "record from an N = 1 run"
side = line["side"]
head = subprocess.run(["git", "-C", str(ROOT), "rev-parse", "--short", "HEAD"], capture_output=True,
                      text=True).stdout.strip()
out = {"_provenance": f"bench.py N=1 on one B200 at {head} (tools/record_n1_digests.py); "
                      "Box-Muller digests change whenever its arithmetic does",
       "cfg2_stats_digest": side["brownian"]["digest"],
       "cfg3_digest": side["box_muller_f64"]["digest"]}
(ROOT / "tests" / "golden" / "gpu_n1_digests.json").write_text(json.dumps(out, indent=1) + "\n")
print(out)
