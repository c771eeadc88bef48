import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r:
        hdr = r; continue
    if hdr is None or len(r) != len(hdr): continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum": continue
    name = d["Kernel Name"].split("(")[0]
    v = float(d["Metric Value"].replace(",", ""))
    unit = d.get("Metric Unit", "")
    if unit in ("nsecond", "ns"): v /= 1000
    elif unit in ("msecond", "ms"): v *= 1000
    agg[name][0] += 1; agg[name][1] += v
tot = sum(a[1] for a in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{k[:60]:60s} {n:6d} {t:10.1f} {t/n:8.1f} {100*t/tot:5.1f}%")
print("total us", round(tot, 1), "launches", sum(a[0] for a in agg.values()))
