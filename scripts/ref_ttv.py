"""CPU time to verdict of the REFERENCE on a BASELINE config (host cores of the
box it runs on), phase by phase as cycheck_main.cpp:88-97 splits it:
    python scripts/ref_ttv.py [config] [restrict 0/1] [early 0/1] [workers ...]
Prints one JSON line (lscpu model, nproc, phases, verdict/MapStats per worker
count). Test infrastructure: drives oracle/_ref only (never the engine)."""
import json
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
restrict = len(sys.argv) > 2 and sys.argv[2] == "1"
early = not (len(sys.argv) > 3 and sys.argv[3] == "0")
workers = [int(x) for x in sys.argv[4:]] or [1, os.cpu_count() or 1]
model = ""
try:
    for line in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines():
        if line.startswith("Model name"):
            model = line.split(":", 1)[1].strip()
except Exception:
    pass
R, F = oracle.Restatement(), oracle.Reference()
p = R.prepare(R.preset(cfg))
t0 = time.perf_counter()
r = F.ttv(p, workers=workers, restrict=restrict, early_exit=early)
print(json.dumps({"config": cfg, "n": int(p.n), "m_log": int(p.m), "restrict": restrict, "early_exit": early,
                  "cpu_model": model, "nproc": os.cpu_count(), "wall_s": round(time.perf_counter() - t0, 1),
                  **r}), flush=True)
