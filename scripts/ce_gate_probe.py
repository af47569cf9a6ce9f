"""Copy-engine behaviour at cfg2 sizes with host enqueue taken out of the
picture: every copy is enqueued while the GPU is held by a sleep kernel, and
the events bracket only the device-side copy work.  Single copies vs N
chunks per direction, both directions concurrently, H2D on one or two
streams."""
import torch
B, z1, z2 = 4096, 1500, 2100
n = z1 + z2 - 1
a = torch.randint(0, 1 << 30, (B, z1 + z2), dtype=torch.int32).pin_memory()
c = torch.empty((B, n), dtype=torch.int32).pin_memory()
da = torch.empty((B, z1 + z2), dtype=torch.int32, device="cuda")
dc = torch.randint(0, 1 << 30, (B, n), dtype=torch.int32, device="cuda")
main = torch.cuda.current_stream()
ss = [torch.cuda.Stream() for _ in range(4)]
mb_in, mb_out = a.numel() * 4 / 1e6, c.numel() * 4 / 1e6


def gated(enqueue, reps=5):
    ts = []
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        torch.cuda._sleep(20_000_000)  # ~10 ms: everything below is enqueued meanwhile
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        for s in ss:
            s.wait_stream(main)
        enqueue()
        for s in ss:
            main.wait_stream(s)
        e1.record(main)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts[1:])


def chunks(nch, total):
    rows = B // nch
    return [slice(i * rows, (i + 1) * rows if i < nch - 1 else B) for i in range(nch)]


def h2d(nch, streams=1):
    def f():
        for i, r in enumerate(chunks(nch, B)):
            with torch.cuda.stream(ss[i % streams]):
                da[r].copy_(a[r], non_blocking=True)
    return f


def d2h(nch):
    def f():
        for r in chunks(nch, B):
            with torch.cuda.stream(ss[2]):
                c[r].copy_(dc[r], non_blocking=True)
    return f


def both(nch, streams=1):
    fi, fo = h2d(nch, streams), d2h(nch)
    def f():
        fi(); fo()
    return f


for nch in (1, 4, 8, 16, 32, 64):
    t1 = gated(h2d(nch)); t2 = gated(d2h(nch)); t3 = gated(both(nch)); t4 = gated(both(nch, 2))
    print(f"nch {nch:3d}: H2D {t1:.3f} ms ({mb_in / t1:.1f} GB/s)  D2H {t2:.3f} ms ({mb_out / t2:.1f} GB/s)"
          f"  both {t3:.3f} ms ({(mb_in + mb_out) / t3:.1f} GB/s)  both/2 H2D streams {t4:.3f} ms", flush=True)


# pipelined shape without kernels: D2H of chunk i waits for H2D of chunk i
def piped(nch, with_kernel=False):
    evs = [torch.cuda.Event() for _ in range(nch)]
    def f():
        for i, r in enumerate(chunks(nch, B)):
            with torch.cuda.stream(ss[0]):
                da[r].copy_(a[r], non_blocking=True)
                evs[i].record(ss[0])
            if with_kernel:
                ss[1].wait_event(evs[i])
                with torch.cuda.stream(ss[1]):
                    dc[r].add_(1)
                    evs[i].record(ss[1])
            ss[2].wait_event(evs[i])
            with torch.cuda.stream(ss[2]):
                c[r].copy_(dc[r], non_blocking=True)
    return f


for nch in (4, 8, 16, 32):
    t1 = gated(piped(nch)); t2 = gated(piped(nch, True))
    print(f"piped nch {nch:3d}: copies {t1:.3f} ms  with a kernel per chunk {t2:.3f} ms", flush=True)
