"""Refresh profiles/traffic.json (read by bench.py for roofline.traffic and
int_pipe.ncu) from a profiling pass: per-step DRAM bytes from the launch
lists (scripts/step_traffic.py) and pipe utilisation from the ncu --set full
summaries.  usage: python scripts/update_traffic.py profiles/r02/ncu"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import statistics  # noqa: E402

from step_traffic import steps  # noqa: E402

d = sys.argv[1]
names = {1: "cfg1_single_1024x1024_p469762049_fft_pad",
         2: "cfg2_tft_batch4096_1500x2100_p2013265921",
         3: "cfg3_fft_pad_batch65536_4096x4096_p998244353",
         4: "cfg4_fft_pad_batch8_2^22x2^22_p2013265921",
         5: "cfg5_three_primes_2^20x2^20_crt"}


def summary(path):
    out = {}
    for line in open(path):
        parts = line.split()
        if len(parts) >= 2:
            out[parts[0] if parts[0] != "stall" else "stall " + parts[1]] = parts[-1]
    return out


t = {}
for c, name in names.items():
    csv_path = os.path.join(d, f"launches_cfg{c}.csv")
    ss = steps(csv_path)
    sig = max(set(tuple(s["kernels"]) for s in ss), key=lambda k: sum(tuple(s["kernels"]) == k for s in ss))
    sel = [s for s in ss if tuple(s["kernels"]) == sig]
    rec = {"kernel": " + ".join(sig),
           "dram_bytes_read": int(statistics.median(s["read"] for s in sel)),
           "dram_bytes_write": int(statistics.median(s["write"] for s in sel)),
           "source": f"{csv_path} (ncu launch list, dram__bytes_read/write summed over one timed "
                     "step, median of the steps; scripts/step_traffic.py)",
           "note": "ncu flushes the caches before each launch: product bytes still dirty in L2 "
                   "when a kernel ends are not counted as writes"}
    full = {2: "prof_cfg2_summary.txt", 3: "prof_cfg3_summary.txt", 4: "prof_cfg4_row_conv_summary.txt",
            5: "prof_cfg5_row_conv_summary.txt"}.get(c)
    if full:
        s = summary(os.path.join(d, full))
        rec["ncu_pipes"] = {
            "fmaheavy_cycles_pct_of_peak": round(float(s["sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"]), 1),
            "alu_cycles_pct_of_peak": round(float(s["sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"]), 1),
            "issue_active_pct": round(float(s["smsp__issue_active.avg.pct_of_peak_sustained_active"]), 1),
            "source": os.path.join(d, full) + (" (row pass: half of the step)" if c == 4 else
                                                 " (one prime's row pass, the largest share of the step)" if c == 5 else "")}
    t[name] = rec
with open("profiles/traffic.json", "w") as f:
    json.dump(t, f, indent=1)
print(json.dumps(t, indent=1)[:1500])
