#!/usr/bin/env python3
"""Condense an ncu launch list (ncu --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file RAW) into

  * a compact CSV (id, kernel, grid, block, gpu_time_ns, dram_read_bytes,
    dram_write_bytes) -> OUT_CSV,
  * per-kernel shares of the summed launch time (printed), and
  * the mean DRAM bytes per launch of the dominant kernel family (template
    arguments stripped) -> profiles/ncu_traffic.json under KEY (the bench's
    roofline.traffic, compared there with the algorithmic bytes per launch).

ncu serialises launches with cold caches, so only SHARES are comparable with
the bench, not absolute times.

    python tools/launch_summary.py RAW.csv OUT_CSV KEY
"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(raw, out_csv, key):
    rows = collections.OrderedDict()
    with open(raw) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rd = csv.reader(lines)
    hdr = next(rd)
    ix = {h: i for i, h in enumerate(hdr)}
    for r in rd:
        if r[0] == "ID":
            continue
        lid = int(r[ix["ID"]])
        d = rows.setdefault(lid, {"kernel": r[ix["Kernel Name"]], "grid": r[ix["Grid Size"]],
                                  "block": r[ix["Block Size"]]})
        d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
    with open(out_csv, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["id", "kernel", "grid", "block", "gpu_time_ns", "dram_read_bytes", "dram_write_bytes"])
        for lid, d in rows.items():
            w.writerow([lid, d["kernel"], d["grid"], d["block"], int(d.get("gpu__time_duration.sum", 0)),
                        int(d.get("dram__bytes_read.sum", 0)), int(d.get("dram__bytes_write.sum", 0))])
    tot = sum(d.get("gpu__time_duration.sum", 0) for d in rows.values())
    by = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for d in rows.values():
        k = d["kernel"].split("(")[0]
        by[k][0] += 1
        by[k][1] += d.get("gpu__time_duration.sum", 0)
        by[k][2] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    print(f"{len(rows)} launches, {tot / 1e3:.1f} us total (serialised, cold)")
    for k, (c, t, b) in sorted(by.items(), key=lambda kv: -kv[1][1]):
        print(f"  {k}: {c} launches, {100 * t / tot:.1f}% of time, mean {t / c / 1e3:.2f} us, "
              f"mean DRAM {b / c / 1e6:.2f} MB/launch")
    fam = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for k, (c, t, b) in by.items():
        f_ = k.split("<")[0].replace("void ", "")
        fam[f_][0] += c
        fam[f_][1] += t
        fam[f_][2] += b
    name, (c, t, b) = max(fam.items(), key=lambda kv: kv[1][1])
    print(f"family {name}: {c} launches, {100 * t / tot:.1f}% of time, mean DRAM {b / c / 1e6:.2f} MB/launch")
    top = (name, c, b / c)
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    data = json.load(open(tp)) if os.path.exists(tp) else {}
    data[key] = int(top[2])
    data["_src_" + key] = (f"{os.path.relpath(out_csv, ROOT)}: mean dram__bytes_read.sum+dram__bytes_write.sum "
                           f"per launch of {top[0]} over {top[1]} launches")
    data.pop("_src", None)
    with open(tp, "w") as f:
        json.dump(data, f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    main(*sys.argv[1:4])
