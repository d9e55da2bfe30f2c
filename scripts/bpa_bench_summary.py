"""One line per JSON line of a `bench.py --bpa` log: python scripts/bpa_bench_summary.py FILE"""
import json
import sys

for ln in open(sys.argv[1]):
    if ln.startswith("{"):
        d = json.loads(ln)
        c = d.get("cpu_baseline") or {}
        print(d["config"]["workload"], f"{d['value']:.1f} Gterms/s", f"{d['ms_per_step']:.2f} ms/step",
              f"kernel {d['roofline']['ms']:.2f} ms", f"frac {d['roofline']['frac']:.3f}",
              f"rel-L2 vs oracle {c.get('rel_l2_of_gpu_vs_oracle_on_sample')}", d["clocks"]["reasons"])
    else:
        print(ln[:300].rstrip())
