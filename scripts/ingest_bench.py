"""Explicit-graph text ingestion: device parse_explicit_graph vs the
reference's (std::getline + istringstream) on the same file.
python scripts/ingest_bench.py [log2 edges]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0912_2555_b200 as eng  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 22
rng = np.random.default_rng(1)
n = 1 << (k - 2)
e = rng.integers(0, n, size=(1 << k, 2), dtype=np.uint32)
acc = np.flatnonzero(rng.random(n) < 0.05)
t0 = time.perf_counter()
body = "\n".join(f"edge {s} {d}" for s, d in e.tolist())
text = f"graph {n}\naccepting {' '.join(map(str, acc.tolist()))}\n{body}\n".encode()
gen_s = time.perf_counter() - t0
out = {"edges": int(len(e)), "bytes": len(text), "text_gen_s": round(gen_s, 2)}
for rep in range(3):
    t0 = time.perf_counter()
    dg = eng.parse_explicit_device(text)
    dev_s = time.perf_counter() - t0
out["device_parse_ms"] = round(dev_s * 1e3, 2)
out["device_GBps"] = round(len(text) / dev_s / 1e9, 2)
assert dg.m == len(e)
try:
    import oracle

    R = oracle.Reference()
    t0 = time.perf_counter()
    rn, racc, re_ = R.parse_explicit(text)
    ref_s = time.perf_counter() - t0
    out["reference_parse_ms"] = round(ref_s * 1e3, 1)
    out["reference_GBps"] = round(len(text) / ref_s / 1e9, 3)
    g = dg.export()
    out["identical"] = bool(rn == g.n and np.array_equal(racc, g.accepting) and np.array_equal(re_, g.edges))
except Exception as ex:  # reference build absent
    out["reference"] = f"unavailable: {ex}"
print(json.dumps(out))
