"""Refreshes profiles/ from a scripts/profile_round.sh run (gpurun_out/):
bench lines, the launch list summary, the ncu --set full details of k_map_run
and the traffic summary bench.py reads. Run here (no GPU needed)."""
import csv
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
TAG = os.environ.get("ROUND_TAG", "r01")


def last_json(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


def main():
    b = last_json(os.path.join(OUT, "bench.log"))
    json.dump(b, open(os.path.join(PROF, f"{TAG}_bench_c2.json"), "w"))
    r = last_json(os.path.join(OUT, "bench_ref.log"))
    json.dump(r, open(os.path.join(PROF, f"{TAG}_bench_reference_c2.json"), "w"))
    # launch list
    rows = list(csv.reader(open(os.path.join(OUT, "launches.csv"))))
    h = next(i for i, x in enumerate(rows) if "Kernel Name" in x)
    hdr = rows[h]
    k, v, u, idc = (hdr.index(x) for x in ("Kernel Name", "Metric Value", "Metric Unit", "ID"))
    agg, lines = defaultdict(lambda: [0, 0.0]), []
    for x in rows[h + 1:]:
        if len(x) <= v:
            continue
        us = float(x[v].replace(",", "")) * {"ms": 1e3, "ns": 1e-3}.get(x[u], 1.0)
        name = x[k].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += us
        lines.append((int(x[idc]), name, us))
    tot = sum(a[1] for a in agg.values())
    with open(os.path.join(PROF, f"{TAG}_launches.txt"), "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv "
                "python bench.py --steps 2 --warmup 3 --no-cpu-baseline\n")
        f.write("# (cold-cache, serialised launches: compare shares, not absolutes). Per-kernel totals:\n")
        for n, (c, t) in sorted(agg.items(), key=lambda y: -y[1][1]):
            f.write(f"{n:48s} launches {c:4d}  total {t / 1e3:10.3f} ms  share {100 * t / tot:5.1f}%\n")
        f.write("\n# k_map_run launches (one per run_map)\n")
        for i, n, t in lines:
            if "k_map_run" in n:
                f.write(f"id {i:4d}  {t / 1e3:9.3f} ms\n")
    # ncu --set full
    rep = os.path.join(OUT, "map_run.ncu-rep")
    det = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
    open(os.path.join(PROF, f"{TAG}_ncu_map_run_full.txt"), "w").write(det)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    hh, units, vals = rr[0], rr[1], rr[2]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
            "launch__grid_size", "launch__block_size"]
    met = {w: [float(vals[hh.index(w)].replace(",", "")), units[hh.index(w)]] for w in want if w in hh}
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
    rd = met["dram__bytes_read.sum"][0] * scale[met["dram__bytes_read.sum"][1]]
    wr = met["dram__bytes_write.sum"][0] * scale[met["dram__bytes_write.sum"][1]]
    summ = {"source": f"profiles/{TAG}_ncu_map_run_full.txt (ncu --set full --clock-control none, k_map_run, "
                      "4th launch of python bench.py --steps 2 --warmup 3 --no-cpu-baseline; config 2)",
            "kernel": "k_map_run", "traffic_bytes_per_launch": int(rd + wr),
            "dram_read_bytes": int(rd), "dram_write_bytes": int(wr), "metrics": met}
    json.dump(summ, open(os.path.join(PROF, "ncu_map_run_summary.json"), "w"), indent=1)
    print(json.dumps({"value": b["value"], "ms": b["ms_per_step"], "e2e": b["e2e"]["value"],
                      "frac": b["roofline"]["frac"], "traffic": summ["traffic_bytes_per_launch"],
                      "ref": r["value"]}))


if __name__ == "__main__":
    main()
