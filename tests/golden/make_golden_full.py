"""Full-size golden fixtures: the REFERENCE (compiled from /root/reference
sources into oracle/_ref/) run on the BASELINE.json configurations at their
stated sizes, on the same seeded logs the device generators produce
(include/cyc_gen.h). Run here, where the reference sources and ~60 GB of RAM
exist (≈40 min on 8 cores):

    python tests/golden/make_golden_full.py [c2 c5 c3 c4 ...]

Writes tests/golden/golden_full.json (merged per config). Recorded per run:
verdict, witness, MapStats (map_engine.cpp:139-162, via ref_run_map, which
replays run_map with the public fixpoint/demote to expose the vectors), the
sha256 digest of the final map vector, every iteration's vector hash
(sum splitmix64((v<<32)|x[v])) and step count, and the snapshot / restricted
snapshot digests (graph.cpp:63-221). tests/test_gpu_full_parity.py compares
the CUDA path against these bit for bit on the GPU box.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

OUT = os.path.join(HERE, "golden_full.json")
WORKERS = os.cpu_count() or 1


def digest(a) -> str:
    h = hashlib.sha256()
    b = np.ascontiguousarray(a).view(np.uint8).reshape(-1)
    for i in range(0, len(b), 1 << 28):
        h.update(b[i:i + (1 << 28)].tobytes())
    return h.hexdigest()[:32]


def log(*a):
    print(time.strftime("%H:%M:%S"), *a, flush=True)


def record(rs, early, acc=None, check=False):
    t0 = time.perf_counter()
    r = rs.run_map(acc, early_exit=early, workers=WORKERS, check_run_map=check)
    rec = {"cycle": r.cycle, "witness": r.witness, "iterations": r.iterations,
           "kernel_calls": r.kernel_calls, "demoted_total": r.demoted_total,
           "final_x_digest": digest(r.final_x),
           "final_x_nonnil": int(np.count_nonzero(r.final_x)),
           "iter_hash": [str(int(h)) for h in r.iter_hash[:512]],
           "iter_steps": [int(s) for s in r.iter_steps[:512]],
           "ref_seconds": round(time.perf_counter() - t0, 1)}
    log(f"  run_map early={early}: cycle={r.cycle} witness={r.witness} it={r.iterations} "
        f"calls={r.kernel_calls} demoted={r.demoted_total} ({rec['ref_seconds']} s)")
    return rec


def snap_digests(rs):
    csr, acc, kept = rs.export()
    return {"n": rs.n, "m": rs.m, "off_digest": digest(csr.off), "col_digest": digest(csr.col),
            "acc_digest": digest(acc)}, kept


# name -> (config index, overrides, runs): runs on the unrestricted snapshot
# ("early"/"full") and on the restricted one ("r_early"/"r_full").
CASES = {
    "c2": (2, {}, ["early", "full"]),
    "c5": (5, {}, ["early"]),
    "c3": (3, {}, ["early", "full", "r_early", "r_full"]),
    "c4": (4, {}, ["r_early", "r_full"]),
}


def run_case(name):
    idx, over, runs = CASES[name]
    R = oracle.Restatement()
    F = oracle.Reference()
    p = R.preset(idx)
    for k, v in over.items():
        setattr(p, k, v)
    R.prepare(p)
    entry = {"config": idx, "overrides": over, "n": int(p.n), "m_log": int(p.m), "workers": WORKERS}
    log(f"{name}: n={p.n} m_log={p.m}")
    t0 = time.perf_counter()
    rs = F.snapshot_gen(p, True)  # reference EdgeLog + build_snapshot (transposed)
    entry["build_snapshot_s_incl_log_fill"] = round(time.perf_counter() - t0, 1)
    tr, _ = snap_digests(rs)
    log(f"  snapshot m={rs.m} ({entry['build_snapshot_s_incl_log_fill']} s)")
    for run in runs:
        if not run.startswith("r_"):
            tr[run] = record(rs, run == "early", check=(name == "c2"))
    if any(r.startswith("r_") for r in runs):
        t0 = time.perf_counter()
        rr = rs.restrict()  # restrict_to_accepting_sccs (graph.cpp:190-221)
        rd, kept = snap_digests(rr)
        rd["kept_digest"] = digest(kept[: rr.n])
        rd["ref_seconds"] = round(time.perf_counter() - t0, 1)
        log(f"  restricted n={rr.n} m={rr.m} ({rd['ref_seconds']} s)")
        for run in runs:
            if run.startswith("r_"):
                rec = record(rr, run == "r_early")
                if rec["cycle"]:
                    rec["witness_original"] = int(kept[rec["witness"]])
                rd[run[2:]] = rec
        tr["restricted"] = rd
        del rr
    entry["transposed"] = tr
    del rs
    return entry


def main():
    names = sys.argv[1:] or list(CASES)
    out = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            out = json.load(f)
    out.setdefault("generator", "tests/golden/make_golden_full.py")
    out.setdefault("reference", "/root/reference/proj @ src/{graph,map_engine,parallel,errors}.cpp "
                   "(graph.hpp:56 patched copy, see oracle/Makefile), driven by oracle/ref_driver.cpp")
    out.setdefault("configs", {})
    for name in names:
        out["configs"][name] = run_case(name)
        with open(OUT, "w") as f:
            json.dump(out, f, indent=1, sort_keys=True)
        log(f"{name} written to {OUT}")


if __name__ == "__main__":
    main()
