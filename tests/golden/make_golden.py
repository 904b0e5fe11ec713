"""Generates the golden fixtures in tests/golden/ by running the REFERENCE
implementation (compiled from /root/reference sources into oracle/_ref/) on
seeded inputs. Run here, where the reference sources exist:

    python tests/golden/make_golden.py

The fixtures travel with the repo; the GPU box never needs /root/reference.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402


def digest(a) -> str:
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def record(rs, acc_words, early):
    r = rs.run_map(None, early_exit=early, workers=1)
    return {
        "cycle": r.cycle, "witness": r.witness, "iterations": r.iterations,
        "kernel_calls": r.kernel_calls, "demoted_total": r.demoted_total,
        "final_x_digest": digest(r.final_x),
        "iter_hash": [int(h) for h in r.iter_hash[:256]],
        "iter_steps": [int(s) for s in r.iter_steps[:256]],
    }, r.final_x


def main():
    F = oracle.Reference()
    R = oracle.Restatement()
    out = {"generator": "tests/golden/make_golden.py", "reference": "/root/reference/proj @ src/"
           "{graph,map_engine,parallel,errors,oracle,owcty}.cpp (graph.hpp:56 patched copy, see oracle/Makefile)",
           "configs": {}, "random": []}
    arrays = {}
    # canonical configurations at full or scaled-down size
    cases = [("c1", 1, {}), ("c2_L16", 2, {"L": 16, "W": 64, "S": 8}),
             ("c5_L16", 5, {"L": 16, "W": 4, "S": 16}), ("c3_s12", 3, {"scale": 12}),
             ("c4_g6", 4, {"grid_bits": 6, "region": 16})]
    for name, idx, over in cases:
        p = R.preset(idx)
        for k, v in over.items():
            setattr(p, k, v)
        R.prepare(p)
        n, edges, accw = R.generate(p)
        entry = {"config": idx, "overrides": over, "n": n, "m_log": int(p.m),
                 "edges_digest": digest(edges), "acc_digest": digest(accw)}
        for tr in (True, False):
            rs = F.snapshot(n, edges, accw, tr)
            csr, acc, _ = rs.export()
            key = "transposed" if tr else "forward"
            entry[key] = {"m": csr.m, "off_digest": digest(csr.off), "col_digest": digest(csr.col)}
            # run_owcty (owcty.cpp:56-87) on the same snapshot
            oc, ow, oit, ofs = rs.run_owcty()
            entry[key]["owcty"] = {"cycle": oc, "witness": ow, "outer_iterations": oit, "final_size": ofs}
            for early in (True, False):
                rec, fx = record(rs, accw, early)
                entry[key]["early" if early else "full"] = rec
                if name in ("c1", "c2_L16"):
                    arrays[f"{name}_{key}_{'early' if early else 'full'}_final_x"] = fx
            rr = rs.restrict()
            rcsr, racc, kept = rr.export()
            entry[key]["restricted"] = {"n": rr.n, "m": rr.m, "kept_digest": digest(kept),
                                        "off_digest": digest(rcsr.off), "col_digest": digest(rcsr.col)}
            for early in (True, False):
                rec, _ = record(rr, racc, early)
                if rec["cycle"]:
                    rec["witness_original"] = int(kept[rec["witness"]])
                entry[key]["restricted"]["early" if early else "full"] = rec
        out["configs"][name] = entry
        print(name, "done", flush=True)
    # small random digraphs with every vector
    rng = np.random.default_rng(0x0912)
    for t in range(60):
        n = int(rng.integers(1, 40))
        m = int(rng.integers(0, 4 * n + 1))
        edges = rng.integers(0, n, size=(m, 2)).astype(np.uint32)
        accb = rng.random(n) < [0.1, 0.3][t % 2]
        rs = F.snapshot(n, edges, accb, True)
        csr, accw, _ = rs.export()
        early_rec, fx_e = record(rs, accw, True)
        full_rec, fx_f = record(rs, accw, False)
        x1, ch1, w1 = rs.step(np.zeros(n, np.uint32))
        out["random"].append({"n": n, "edges": edges.tolist(), "accepting": np.flatnonzero(accb).tolist(),
                              "row_offsets": csr.off.tolist(), "col_indices": csr.col.tolist(),
                              "step1": x1.tolist(), "step1_changed": ch1,
                              "early": early_rec, "full": full_rec,
                              "final_x_early": fx_e.tolist(), "final_x_full": fx_f.tolist(),
                              "scc_cycle": rs.scc_verdict()})
    # explicit-graph texts through the reference's parse_explicit_graph
    import base64
    sys.path.insert(0, os.path.dirname(HERE))
    import explicit_cases

    out["explicit"] = []
    for text in explicit_cases.cases():
        rec = {"text_b64": base64.b64encode(text).decode()}
        try:
            n, acc, e = F.parse_explicit(text)
            rec["n"], rec["accepting"], rec["edges"] = n, acc.tolist(), e.tolist()
        except oracle.RefParseError as ex:
            rec["error"] = str(ex)
        out["explicit"].append(rec)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "golden_vectors.npz"), **arrays)
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
