"""Fig. 3 methodology with device time: per n, fft_pad vs tft ns per product
of one batched conv_batch call (CUDA events, median of reps), inputs resident
on the GPU, B*L ~ 2^25 positions per call so launch latency does not count.
CSV in the reference sweep schema (cli.py:195).

    python scripts/fig3_device.py --min 4000 --max 4300 --step 12 -o out.csv
"""
import argparse
import statistics
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1609_01010_b200 as mc  # noqa: E402
from paper_1609_01010_b200.transform import OpCounters  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--min", type=int, required=True)
ap.add_argument("--max", type=int, required=True)
ap.add_argument("--step", type=int, default=1)
ap.add_argument("--prime", type=int, default=998244353)
ap.add_argument("--reps", type=int, default=15)
ap.add_argument("--positions", type=int, default=1 << 25)
ap.add_argument("-o", "--output", required=True)
args = ap.parse_args()

p = args.prime
fp = mc.FourierPrime.from_modulus(p)
rows = ["n,engine,threads,nanos_median,nanos_mean,butterflies,pointwise_muls"]
g = torch.Generator(device="cuda").manual_seed(1)
for n in range(args.min, args.max + 1, args.step):
    z1 = (n + 1) // 2
    z2 = n + 1 - z1
    L = 1 << (n - 1).bit_length()
    B = max(16, args.positions // L)
    a = torch.randint(0, p, (B, z1), generator=g, device="cuda", dtype=torch.int64).to(torch.int32)
    b = torch.randint(0, p, (B, z2), generator=g, device="cuda", dtype=torch.int64).to(torch.int32)
    for eng in ("fft_pad", "tft"):
        cnt = OpCounters()
        mc.conv_batch(a[:1], b[:1], fp, engine=eng, counters=cnt)
        out = mc.conv_batch(a, b, fp, engine=eng)
        ts = []
        for _ in range(args.reps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            mc.conv_batch(a, b, fp, engine=eng, out=out)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e6 / B)
        rows.append(f"{n},{eng},1,{statistics.median(ts):.2f},{statistics.fmean(ts):.2f},"
                    f"{cnt.butterflies},{cnt.pointwise_muls}")
with open(args.output, "w") as fh:
    fh.write("\n".join(rows) + "\n")
print(f"wrote {len(rows) - 1} rows to {args.output}")
