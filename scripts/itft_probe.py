"""itft (L = 4096, n = 3599) on 4096 rows through mc_itft: device time."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1609_01010_b200 import _native
lib = _native.lib()
p, K, n, B = 2013265921, 12, 3599, 4096
x = torch.randint(0, p, (B, n), dtype=torch.int64).to(torch.int32).cuda()
y = torch.empty_like(x)
st = torch.cuda.current_stream()
f = lambda: _native.check(lib.mc_itft(x.data_ptr(), y.data_ptr(), n, K, B, p, st.cuda_stream))
f(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(10): f()
e1.record(st); torch.cuda.synchronize()
print("itft ms", e0.elapsed_time(e1) / 10)
