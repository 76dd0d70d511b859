"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel."""
import csv
import re
import sys
from collections import defaultdict


def summarize(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = defaultdict(lambda: [0, 0.0])
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        n = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "")
        n = n.replace("cpd::(anonymous namespace)::", "").replace("cpd::<unnamed>::", "").replace("<unnamed>::", "")
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(d["Metric Unit"], 1e-3)
        agg[n][0] += 1
        agg[n][1] += float(d["Metric Value"].replace(",", "")) * scale
    return agg


if __name__ == "__main__":
    agg = summarize(sys.argv[1])
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':52s} {'launches':>8s} {'total_us':>12s} {'us/launch':>10s} {'share':>7s}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:52]:52s} {v[0]:8d} {v[1]:12.1f} {v[1] / v[0]:10.1f} {100 * v[1] / tot:6.2f}%")
