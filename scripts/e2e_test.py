"""e2e (host pinned buffers) timing of conv_batch for several chunk sizes."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1609_01010_b200 as mc
from paper_1609_01010_b200 import _native, _tensors
p, z1, z2, B = 2013265921, 1500, 2100, 4096
n = z1 + z2 - 1
a = torch.randint(0, p, (B, z1), dtype=torch.int64).to(torch.int32).pin_memory()
b = torch.randint(0, p, (B, z2), dtype=torch.int64).to(torch.int32).pin_memory()
c = torch.empty((B, n), dtype=torch.int32).pin_memory()
st = torch.cuda.current_stream()
for chunk in (0, 128, 256, 512, 1024, 4096):
    def run():
        _native.check(_native.lib().mc_conv_host_async(1, a.data_ptr(), z1, z1, b.data_ptr(), z2, z2,
                      c.data_ptr(), n, B, p, chunk, st.cuda_stream))
    run(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): run()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"chunk {chunk:5d}: {ms:.3f} ms/step  {B / ms * 1e3 / 1e6:.3f} M products/s  "
          f"{4 * B * (z1 + z2 + n) / ms / 1e6:.1f} GB/s total")
