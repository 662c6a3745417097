"""Mean duration per kernel from an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import collections
import csv
import sys

for path in sys.argv[1:]:
    hdr, agg = None, collections.defaultdict(list)
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                agg[d["Kernel Name"].split("(")[0][-48:]].append(float(d["Metric Value"].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    print(path)
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"  {k:48s} n={len(v):3d} mean={sum(v) / len(v) / 1e3:9.2f} us  share={sum(v) / tot:6.1%}")
