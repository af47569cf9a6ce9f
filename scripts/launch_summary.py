"""Aggregate an ncu --csv launch list: per kernel name, count and mean metrics."""
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ik, im, iv, iu = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
iid = h.index("ID")
per = collections.defaultdict(dict)
for r in rows[1:]:
    per[r[iid]][r[im]] = (r[iv].replace(",", ""), r[iu]); per[r[iid]]["_k"] = (r[ik][:60], "")
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for lid, d in per.items():
    for m, (v, u) in d.items():
        if m != "_k":
            try: agg[d["_k"][0]][m].append(float(v))
            except ValueError: pass
for k, ms in agg.items():
    n = len(ms.get("gpu__time_duration.sum", []))
    s = " ".join(f"{m.split('__')[1][:28]}={sum(v)/len(v):.4g}" for m, v in sorted(ms.items()))
    print(f"{n:3d}x {k:60s} {s}")
