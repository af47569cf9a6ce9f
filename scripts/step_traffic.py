"""Per-step DRAM traffic of our kernels from an ncu launch list with
gpu__time_duration / dram__bytes_{read,write}: steps are delimited by the
L2-flush fill kernel bench.py runs before every timed step."""
import csv, json, statistics, sys

def steps(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ik, im, iv, iid = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = {}
    for r in rows[1:]:
        d = per.setdefault(int(r[iid]), {"k": r[ik]})
        d[r[im]] = float(r[iv].replace(",", ""))
    out, cur = [], None
    for i in sorted(per):
        d = per[i]
        if "FillFunctor" in d["k"]:
            if cur:
                out.append(cur)
            cur = {"kernels": [], "read": 0.0, "write": 0.0, "ns": 0.0}
        elif cur is not None and "mc::" in d["k"]:
            cur["kernels"].append(d["k"].split("(")[0].replace("void ", ""))
            cur["read"] += d.get("dram__bytes_read.sum", 0)
            cur["write"] += d.get("dram__bytes_write.sum", 0)
            cur["ns"] += d.get("gpu__time_duration.sum", 0)
    if cur:
        out.append(cur)
    return [s for s in out if s["kernels"]]

if __name__ == "__main__":
    for path in sys.argv[1:]:
        ss = steps(path)
        sig = max(set(tuple(s["kernels"]) for s in ss), key=lambda k: sum(tuple(s["kernels"]) == k for s in ss))
        sel = [s for s in ss if tuple(s["kernels"]) == sig]
        print(json.dumps({"file": path, "steps": len(sel), "kernels": list(sig),
                          "read": statistics.median(s["read"] for s in sel),
                          "write": statistics.median(s["write"] for s in sel),
                          "us": statistics.median(s["ns"] for s in sel) / 1e3}))
