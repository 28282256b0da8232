#!/usr/bin/env python3
"""Copy an evidence run (tools/gpu_evidence.sh -> gpurun_out/ev/) into
profiles/: bench lines as bench_r01_final_*.json, condensed launch lists and
traffic, ncu --set full summaries, and the bench table of profiles/README.md.

    python tools/update_profiles.py [gpurun_out/ev]
"""
import glob
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")


def main(ev):
    for f in glob.glob(os.path.join(PROF, "bench_r01_final_*.json")):
        os.unlink(f)
    for f in sorted(glob.glob(os.path.join(ev, "bench_*.json"))):
        tag = os.path.basename(f)[len("bench_"):-len(".json")]
        shutil.copy(f, os.path.join(PROF, f"bench_r01_final_{tag}.json"))
    for tag, key in (("7b", "llama2-7b-decode:n1"), ("7bfused", "llama2-7b-decode-fused-qkv-gateup:n1")):
        raw = os.path.join(ev, f"launches_{tag}.csv")
        if os.path.exists(raw):
            out = os.path.join(PROF, "ncu_launches_r01_7b_decode" + ("_fused" if tag == "7bfused" else "") + ".csv")
            subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launch_summary.py"), raw, out, key], check=True)
    reps = [os.path.join(ev, "prof_gemv_4096x11008_n1.ncu-rep"), os.path.join(ev, "prof_tc_4096x11008_n512.ncu-rep")]
    lines = []
    for r in reps:
        if os.path.exists(r):
            lines.append(f"== {os.path.basename(r)[:-len('.ncu-rep')]}")
            lines.append(subprocess.run(["bash", os.path.join(ROOT, "tools", "ncu_summary.sh"), r],
                                        capture_output=True, text=True).stdout.rstrip())
    if lines:
        with open(os.path.join(PROF, "ncu_full_r01_summary.txt"), "w") as fh:
            fh.write("\n".join(lines) + "\n")
    rows = []
    for f in sorted(glob.glob(os.path.join(PROF, "bench_r01_final_*.json"))):
        d = json.load(open(f))
        rows.append((os.path.basename(f), d["config"].get("workload"), d["value"], d["unit"], d.get("hbm_gbs"),
                     d.get("tflops"), d.get("ms_per_step"), (d.get("roofline") or {}).get("frac"),
                     (d.get("e2e") or {}).get("value")))
    p = os.path.join(PROF, "README.md")
    s = open(p).read()
    a = s.index("| file | workload |")
    b = s.index("Other files:")
    tab = ["| file | workload | value | unit | HBM GB/s | TFLOP/s | ms/step | roofline frac | e2e |",
           "|---|---|---|---|---|---|---|---|---|"]
    tab += ["| " + " | ".join(str(x) for x in r) + " |" for r in rows]
    open(p, "w").write(s[:a] + "\n".join(tab) + "\n\n" + s[b:])
    print("\n".join(tab))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "ev"))
