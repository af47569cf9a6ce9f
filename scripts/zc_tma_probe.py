"""Does the bulk-copy (TMA) row prefetch work from page-locked host memory?
Zero-copy conv_batch with MC_ZC_TMA=1 vs the device-resident result."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1609_01010_b200 as mc
p, B, z1, z2 = 2013265921, 4096, 1500, 2100
g = torch.Generator().manual_seed(1)
a = torch.randint(0, p, (B, z1), generator=g, dtype=torch.int64).to(torch.int32)
b = torch.randint(0, p, (B, z2), generator=g, dtype=torch.int64).to(torch.int32)
want = mc.conv_batch(a.cuda(), b.cuda(), p, engine="tft").cpu()
ah, bh = a.pin_memory(), b.pin_memory()
ch = torch.empty((B, z1 + z2 - 1), dtype=torch.int32).pin_memory()
mc.conv_batch(ah, bh, p, engine="tft", out=ch)
print("equal", torch.equal(ch, want), flush=True)
torch.cuda.synchronize()
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(10):
    mc.conv_batch(ah, bh, p, engine="tft", out=ch)
e1.record(st); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"zero copy (MC_ZC_TMA={os.environ.get('MC_ZC_TMA', '')}): {ms:.3f} ms/step  {B / ms / 1e3:.3f} M products/s", flush=True)
