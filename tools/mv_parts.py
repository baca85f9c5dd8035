"""Matvec diagnostics (tools): time h2_matvec of the C2 factor L under H2_MV_PART / H2_MV_WALK
variants, each in a fresh process (the switches are read once).  Writes one JSON line per variant."""
import json
import os
import subprocess
import sys

N = sys.argv[1] if len(sys.argv) > 1 else "512"
for name, env in (("full", {}), ("far_only", {"H2_MV_PART": "1"}), ("near_only", {"H2_MV_PART": "2"}),
                  ("fwd_only", {"H2_MV_PART": "3"}), ("fwd_couple", {"H2_MV_PART": "4"}),
                  ("fwd_couple_bwdsub", {"H2_MV_PART": "5"})):
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "tools/time_matvec.py", N, "factor"], env=e, capture_output=True, text=True)
    line = [l for l in r.stdout.splitlines() if l.startswith("{")]
    print(json.dumps({"variant": name, **(json.loads(line[-1]) if line else {"error": r.stderr[-300:]})}), flush=True)
