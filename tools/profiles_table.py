"""Markdown table of the bench lines under profiles/r02/ (profiles/README.md).
    python tools/profiles_table.py"""
import glob
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
print("| file | workload | value | unit | HBM GB/s | TFLOP/s | ms/step | roofline frac | e2e | clocks |")
print("|---|---|---|---|---|---|---|---|---|---|")
for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "r02", "bench_r02_*.json"))):
    d = json.load(open(f))
    name = os.path.basename(f)
    if d.get("impl") == "reference":
        print(f"| {name} | reference (CPU oracle) | {d['value']} | {d['unit']} | – | – | {d['ms_per_step']} (one sample) "
              f"| – | – | – |")
        continue
    c = d["config"]
    r = d["roofline"]
    ck = d.get("clocks", {})
    print(f"| {name} | {c['workload']} n={c['tokens_per_step']} | {d['value']} | {d['unit']} | {d['hbm_gbs']} "
          f"| {d['tflops']} | {d['ms_per_step']} | {r['frac']} ({r['bound']}) | {d['e2e']['value']} "
          f"| {ck.get('sm_mhz')} MHz {','.join(ck.get('reasons', [])) or '-'} |")
