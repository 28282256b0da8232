#!/usr/bin/env python3
"""Summarise sweep JSONL files (tools/sweep.py) as markdown tables.

    python tools/summarize_sweep.py profiles/sweep_c3_r01.jsonl [...]

Per (K, N): n, variant/tile/split chosen, microseconds per call (back-to-back
in a CUDA graph over >= 4x L2 of distinct weight copies), algorithmic GB/s
and TFLOP/s, and the fraction of the measured peaks (MEASURED_PEAKS.json).
"""
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["hbm_gbs"], d["bf16_tflops"]
    return 6650.0, 1590.0


def main(paths):
    hbm, tf = peaks()
    rows = []
    for p in paths:
        for line in open(p):
            r = json.loads(line)
            if "error" not in r:
                rows.append(r)
    by = collections.defaultdict(list)
    for r in rows:
        by[(r["K"], r["N"])].append(r)
    for (K, N), rs in by.items():
        print(f"\n#### K={K} N={N}  (q4 weight {(K * N // 2 + K // 32 * N * 2) / 1e6:.2f} MB)\n")
        print("| n | variant | schedule | µs | GB/s | TFLOP/s | % HBM | % TC |")
        print("|---|---|---|---|---|---|---|---|")
        for r in sorted(rs, key=lambda r: (r["n"], r["variant"])):
            s = r["sched"]
            sched = f"{s['variant']}/{s['tile']}/s{s['split_k']}" if r["variant"] == "auto" else "-"
            print(f"| {r['n']} | {r['variant']} | {sched} | {r['us']:.2f} | {r['GBps']:.0f} | {r['TFLOPS']:.1f} | "
                  f"{100 * r['GBps'] / hbm:.0f} | {100 * r['TFLOPS'] / tf:.0f} |")


if __name__ == "__main__":
    main(sys.argv[1:])
