"""e2e pipeline shapes at cfg2 sizes (pinned host buffers, whole-batch device
staging, H2D / kernel / D2H per chunk on three streams with events): uniform
vs ramped chunk schedules, against zero copy (conv_batch on pinned tensors)."""
import torch
import paper_1609_01010_b200 as mc
from paper_1609_01010_b200 import _native, _tensors

p, B, z1, z2 = 2013265921, 4096, 1500, 2100
n = z1 + z2 - 1
lib = _native.lib()
a = torch.empty((B, z1), dtype=torch.int32, device="cuda")
b = torch.empty((B, z2), dtype=torch.int32, device="cuda")
_native.check(lib.mc_gen_u32(2, 0, 0, B, z1, p, a.data_ptr(), z1, 0))
_native.check(lib.mc_gen_u32(2, 1, 0, B, z2, p, b.data_ptr(), z2, 0))
want = mc.conv_batch(a, b, p, engine="tft")
a_h, b_h = a.cpu().pin_memory(), b.cpu().pin_memory()
c_h = torch.empty((B, n), dtype=torch.int32).pin_memory()
da, db, dc = torch.empty_like(a), torch.empty_like(b), torch.empty_like(want)
s_in, s_cmp, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
main = torch.cuda.current_stream()


def pipe(sched):
    bounds, r = [], 0
    for k in sched:
        bounds.append((r, r + k)); r += k
    assert r == B
    ev_in = [torch.cuda.Event() for _ in bounds]
    ev_c = [torch.cuda.Event() for _ in bounds]
    def fn():
        s_in.wait_stream(main); s_cmp.wait_stream(main); s_out.wait_stream(main)
        for i, (r0, r1) in enumerate(bounds):
            with torch.cuda.stream(s_in):
                da[r0:r1].copy_(a_h[r0:r1], non_blocking=True)
                db[r0:r1].copy_(b_h[r0:r1], non_blocking=True)
                ev_in[i].record(s_in)
            s_cmp.wait_event(ev_in[i])
            _native.check(lib.mc_conv_tft(da[r0].data_ptr(), z1, z1, db[r0].data_ptr(), z2, z2,
                                          dc[r0].data_ptr(), n, r1 - r0, p, s_cmp.cuda_stream))
            ev_c[i].record(s_cmp)
            s_out.wait_event(ev_c[i])
            with torch.cuda.stream(s_out):
                c_h[r0:r1].copy_(dc[r0:r1], non_blocking=True)
        main.wait_stream(s_out)
        main.synchronize()
    return fn


def zc():
    mc.conv_batch(a_h, b_h, p, engine="tft", out=c_h)


def timeit(fn, reps=8):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main); fn(); e1.record(main); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


scheds = {
    "uniform8": [512] * 8,
    "uniform16": [256] * 16,
    "ramp_a": [64, 128, 256, 512, 512, 512, 512, 512, 512, 352, 128, 64, 32],
    "ramp_b": [128, 256, 512, 768, 768, 768, 512, 256, 128],
    "ramp_c": [32, 64, 128, 256, 512, 1024, 1024, 512, 256, 128, 96, 48, 16],
    "ramp_d": [64, 192, 448, 704, 704, 704, 704, 384, 128, 64],
}
t = timeit(zc); print(f"zero copy     {t:.3f} ms  {B / t * 1e3 / 1e6:.2f} M products/s")
assert torch.equal(c_h.cuda(), want)
for name, s in scheds.items():
    c_h.zero_()
    t = timeit(pipe(s)); ok = torch.equal(c_h.cuda(), want)
    print(f"{name:12s}  {t:.3f} ms  {B / t * 1e3 / 1e6:.2f} M products/s  ok={ok}")
