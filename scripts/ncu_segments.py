"""Per-barrier-segment instruction/stall breakdown of an ncu source page."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]; data = rows[2:]
iS = h.index("Warp Stall Sampling (All Samples)"); iE = h.index("Instructions Executed"); iSrc = h.index("Source")
tot = sum(int(r[iS]) for r in data if r[iS].isdigit())
seg = 0; segs = {}
for i, r in enumerate(data):
    s = int(r[iS]) if r[iS].isdigit() else 0
    e = int(r[iE]) if r[iE].isdigit() else 0
    d = segs.setdefault(seg, [0, 0, 0, i, {}]); d[0] += s; d[1] += e; d[2] += 1
    op = r[iSrc].split()[0] if r[iSrc].split() else ""
    if op.startswith("@"):
        op = r[iSrc].split()[1]
    d[4][op] = d[4].get(op, 0) + e
    if 'BAR.SYNC' in r[iSrc] or 'EXIT' in r[iSrc]:
        seg += 1
for k, v in segs.items():
    if v[1] == 0: continue
    top = sorted(v[4].items(), key=lambda x: -x[1])[:6]
    print(f"seg {k:2d} line {v[3]:5d} n {v[2]:5d} samples {100*v[0]/tot:5.1f}% exec {v[1]/1e6:7.2f}M  " +
          " ".join(f"{o}:{c/1e6:.2f}" for o, c in top))
