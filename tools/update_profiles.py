"""Copy one evidence run (tools/evidence_r01.sh -> gpurun_out/ev/) into profiles/.

    python tools/update_profiles.py [--ev gpurun_out/ev]

Writes the bench JSON lines (profiles/bench_r01_*.json, bench_ref_r01.json), the layer sweep,
the logits timings, the C2 launch list, and refreshes profiles/ncu_summary.json from the
`ncu --set full` captures (durations, DRAM bytes per launch / per stream-sample, pipe
utilisation).  Needs the `ncu` CLI to read the .ncu-rep files.  Prints what it changed;
the prose in profiles/README.md and ncu_r01_final.md is edited by hand.
"""
import argparse
import collections
import csv
import io
import json
import os
import shutil
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")


def last_json(path):
    lines = [l for l in open(path) if l.startswith("{")]
    return lines[-1] if lines else None


def ncu_raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return {}
    units = dict(zip(rows[0], rows[1]))
    vals = dict(zip(rows[0], rows[2]))

    def num(k, scale_to=None):
        v, u = vals.get(k), units.get(k, "")
        if v in (None, ""):
            return None
        x = float(v.replace(",", ""))
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0,
                "usecond": 1e-3, "msecond": 1.0, "nsecond": 1e-6}.get(u, 1.0)
        return x * mult

    return {"kernel": vals.get("Kernel Name"),
            "ms": num("gpu__time_duration.sum"),
            "dram_read": num("dram__bytes_read.sum"), "dram_write": num("dram__bytes_write.sum"),
            "fma_avg": num("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
            "fma_max": num("sm__pipe_fma_cycles_active.max.pct_of_peak_sustained_active"),
            "tc_avg": num("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ev", default=os.path.join(ROOT, "gpurun_out", "ev"))
    a = ap.parse_args()
    ev = a.ev
    for src, dst in [("bench_c2", "bench_r01_c2"), ("bench_c2_approx", "bench_r01_c2_approx"),
                     ("bench_c2_cond", "bench_r01_c2_cond"), ("bench_c3", "bench_r01_c3"),
                     ("bench_c4", "bench_r01_c4"), ("bench_c4_tf32", "bench_r01_c4_tf32"),
                     ("bench_c5", "bench_r01_c5_8k"), ("bench_ref", "bench_ref_r01")]:
        p = os.path.join(ev, src + ".json")
        if os.path.exists(p) and last_json(p):
            open(os.path.join(PROF, dst + ".json"), "w").write(last_json(p))
            print("wrote", dst, json.loads(last_json(p)).get("value"))
    for src, dst in [("sweep.log", "sweep_r01_layers.txt"), ("launches_c2.csv", "launches_r01_c2.csv"),
                     ("gpu_tests.log", "gpu_tests_r01.txt")]:
        p = os.path.join(ev, src)
        if os.path.exists(p):
            if src == "gpu_tests.log":
                open(os.path.join(PROF, dst), "w").write(open(p).read().strip().splitlines()[-1] + "\n")
            else:
                shutil.copy(p, os.path.join(PROF, dst))
            print("wrote", dst)
    for src, dst in [("logits.json", "logits_r01_c2.json"), ("logits_c3.json", "logits_r01_c3.json"),
                     ("logits_c4.json", "logits_r01_c4.json")]:
        p = os.path.join(ev, src)
        if os.path.exists(p) and last_json(p):
            open(os.path.join(PROF, dst), "w").write(last_json(p))
            print("wrote", dst)

    sp = os.path.join(PROF, "ncu_summary.json")
    d = json.load(open(sp))
    caps = {"C2": ("cluster_c2.ncu-rep", None), "C3": ("cluster_c3.ncu-rep", None),
            "C4": ("batch_c4.ncu-rep", 200 * 256), "C5": ("batch_c5.ncu-rep", 100 * 896),
            "logits_parallel_C2": ("parallel_c2.ncu-rep", None)}
    for key, (rep, stream_samples) in caps.items():
        rp = os.path.join(ev, rep)
        if not os.path.exists(rp):
            continue
        r = ncu_raw(rp)
        if not r.get("ms"):
            continue
        e = d.setdefault(key, {})
        if key.startswith("logits"):
            e["gpu__time_duration_us"] = round(r["ms"] * 1e3, 2)
        else:
            e["gpu__time_duration_ms"] = round(r["ms"], 3)
        e["dram_bytes_read"] = int(r["dram_read"] or 0)
        e["dram_bytes_write"] = int(r["dram_write"] or 0)
        if stream_samples:
            e["dram_bytes_per_stream_sample"] = round((e["dram_bytes_read"] + e["dram_bytes_write"]) / stream_samples)
        elif key == "C2":
            e["dram_bytes_per_launch"] = e["dram_bytes_read"] + e["dram_bytes_write"]
        if r.get("fma_avg") is not None and key in ("C2", "C3"):
            e["sm__pipe_fma_cycles_active_pct_of_peak_active"] = {"avg_over_148_sms": round(r["fma_avg"], 2),
                                                                   "max_sm": round(r["fma_max"], 1)}
        if r.get("tc_avg") is not None and key not in ("C2", "C3"):
            e["sm__pipe_tc_cycles_active_pct_of_peak_active_avg"] = round(r["tc_avg"], 2)
        print("ncu", key, round(r["ms"], 3), "ms")
    lp = os.path.join(ev, "launches_c2.csv")
    if os.path.exists(lp):
        rows = [r for r in csv.reader(l for l in open(lp) if l.startswith('"'))]
        agg = collections.OrderedDict()
        for r in rows[1:]:
            x = dict(zip(rows[0], r))
            k = x["Kernel Name"].split("(")[0]
            v = agg.setdefault(k, [0, 0.0])
            v[0] += 1
            v[1] += float(x["Metric Value"]) / 1e6
        tot = sum(v[1] for v in agg.values())
        d["launch_list_C2"] = {k: {"launches": v[0], "ms": round(v[1], 3), "share_pct": round(100 * v[1] / tot, 3)}
                               for k, v in agg.items()}
    json.dump(d, open(sp, "w"), indent=1)
    print("wrote ncu_summary.json")


if __name__ == "__main__":
    main()
