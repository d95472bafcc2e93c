"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum,launch__grid_size --csv) by kernel.

    python scripts/launch_list.py gpurun_out/launches.csv profiles/rNN_launches.json "<command>" [skip]

``skip`` drops the first N launches (the warm-up step).  ncu serialises kernels, so the
per-kernel times have no stream overlap: compare SHARES with the bench, not absolute time.
"""

import csv
import io
import json
import sys


def main(src, out, command, skip=0):
    txt = open(src).read()
    start = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[start:])))
    by_id = {}
    for r in rows:
        k = by_id.setdefault(r["ID"], {"name": r["Kernel Name"]})
        unit = r["Metric Unit"]
        val = float(r["Metric Value"].replace(",", ""))
        if r["Metric Name"] == "gpu__time_duration.sum":
            k["ns"] = val * {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "second": 1e9, "s": 1e9}[unit]
        elif r["Metric Name"] == "launch__grid_size":
            k["grid"] = int(val)
    launches = [by_id[i] for i in sorted(by_id, key=int)][int(skip):]
    agg = {}
    for k in launches:
        name = k["name"].split("(")[0][:90]
        a = agg.setdefault(name, {"name": name, "launches": 0, "us": 0.0})
        a["launches"] += 1
        a["us"] += k.get("ns", 0.0) / 1e3
    total = sum(a["us"] for a in agg.values())
    kernels = sorted(agg.values(), key=lambda a: -a["us"])
    for a in kernels:
        a["share"] = a["us"] / total
    json.dump({"source": command, "launches": len(launches), "total_us": total, "kernels": kernels},
              open(out, "w"), indent=1)
    for a in kernels[:25]:
        print(f'{a["share"]*100:6.2f}%  {a["us"]:10.1f} us  {a["launches"]:5d}  {a["name"]}')


if __name__ == "__main__":
    main(*sys.argv[1:])
