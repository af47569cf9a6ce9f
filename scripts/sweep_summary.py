"""Summarise Fig. 3 sweep CSVs: per n, fft_pad vs tft ns per product and the gain."""
import csv
import sys

for path in sys.argv[1:]:
    d = {}
    for r in csv.DictReader(open(path)):
        d.setdefault(int(r["n"]), {})[r["engine"]] = float(r["nanos_median"])
    print(path)
    worst = None
    for n, v in sorted(d.items()):
        if "fft_pad" in v and "tft" in v and v["fft_pad"] > 0:
            g = 1 - v["tft"] / v["fft_pad"]
            worst = g if worst is None else min(worst, g)
            print(f"  n={n:6d} fft_pad {v["fft_pad"]:8.1f} tft {v["tft"]:8.1f}  tft gain {100 * g:5.1f}%")
    print(f"  worst tft gain {100 * worst:.1f}%")
