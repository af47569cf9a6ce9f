"""Cost of stream memory operations between chunked copy-engine copies
(cfg2 sizes): H2D chunks with/without cuStreamWriteValue32 after each, D2H
chunks with/without an (already satisfied) cuStreamWaitValue32 before each,
and both directions together."""
import torch
from cuda.bindings import driver as drv

B, z1, z2 = 4096, 1500, 2100
n = z1 + z2 - 1
a = torch.randint(0, 1 << 30, (B, z1 + z2), dtype=torch.int32).pin_memory()
c = torch.empty((B, n), dtype=torch.int32).pin_memory()
da = torch.empty((B, z1 + z2), dtype=torch.int32, device="cuda")
dc = torch.randint(0, 1 << 30, (B, n), dtype=torch.int32, device="cuda")
flags = torch.zeros(1024, dtype=torch.int32, device="cuda")
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
main = torch.cuda.current_stream()
W = drv.CUstreamWriteValue_flags.CU_STREAM_WRITE_VALUE_DEFAULT
G = drv.CUstreamWaitValue_flags.CU_STREAM_WAIT_VALUE_GEQ
F = drv.CUstreamWriteValue_flags.CU_STREAM_WRITE_VALUE_NO_MEMORY_BARRIER


def timeit(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for _ in range(reps):
        fn()
    e1.record(main)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def run(nch, h2d=True, d2h=False, write=False, wait=False, wflag=W):
    rows = B // nch
    def fn():
        s_in.wait_stream(main); s_out.wait_stream(main)
        for i in range(nch):
            r = slice(i * rows, (i + 1) * rows)
            if h2d:
                with torch.cuda.stream(s_in):
                    da[r].copy_(a[r], non_blocking=True)
                if write:
                    drv.cuStreamWriteValue32(s_in.cuda_stream, flags.data_ptr() + 4 * i, 1, wflag)
            if d2h:
                if wait:
                    drv.cuStreamWaitValue32(s_out.cuda_stream, flags.data_ptr() + 4 * 1000, 0, G)
                with torch.cuda.stream(s_out):
                    c[r].copy_(dc[r], non_blocking=True)
        main.wait_stream(s_in); main.wait_stream(s_out)
    return fn


for nch in (8, 16, 32):
    for kw in (dict(), dict(write=True), dict(write=True, wflag=F)):
        t = timeit(run(nch, **kw)); print(f"H2D  {nch:2d} {str(kw):40s} {t:.3f} ms")
    for kw in (dict(h2d=False, d2h=True), dict(h2d=False, d2h=True, wait=True)):
        t = timeit(run(nch, **kw)); print(f"D2H  {nch:2d} {str(kw):40s} {t:.3f} ms")
    for kw in (dict(d2h=True), dict(d2h=True, write=True, wait=True)):
        t = timeit(run(nch, **kw)); print(f"BOTH {nch:2d} {str(kw):40s} {t:.3f} ms")
