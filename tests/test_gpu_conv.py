"""GPU parity of the fused convolution engines (configs 1-3 and the
reference's own small-size sweeps) against the C oracle and the reference's
golden fixtures.  Bit-exact: integer residues must be identical."""

import numpy as np
import pytest
import torch

from conftest import P1, P2, P3

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_1609_01010_b200 as mc
    from gpu_helpers import eval_check, gen_device, sha_row, to_u32_np


def _conv(a, b, p, engine):
    at = torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32)).cuda()
    bt = torch.from_numpy(np.ascontiguousarray(b, dtype=np.uint32).view(np.int32)).cuda()
    return to_u32_np(mc.conv_batch(at, bt, p, engine=engine))


@pytest.mark.parametrize("engine", ["fft_pad", "tft"])
def test_golden_small_convs(golden_small, engine):
    for c in golden_small["convs"]:
        p = c["p"]
        if c.get("tag") == "all_p_minus_1":
            u = np.full(c["z1"], p - 1)
            v = np.full(c["z2"], p - 1)
        else:
            u, v = np.array(c["u"]), np.array(c["v"])
        got = _conv(u[None], v[None], p, engine)[0]
        assert got.tolist() == c[engine], (p, len(u), len(v), engine)


def test_kats(golden_small):
    k = golden_small["kats"]
    for c in k["conv17"]:
        for eng in ("fft_pad", "tft"):
            got = _conv(np.array([c["u"]]), np.array([c["v"]]), 17, eng)[0]
            assert got.tolist() == c[eng]


@pytest.mark.parametrize("engine", ["fft_pad", "tft"])
@pytest.mark.parametrize("p", [P2, P3])
def test_sweep_64x64_vs_oracle(orc, engine, p):
    """conv_tft vs schoolbook for all 64x64 length pairs
    (reference tests/test_convolve.py:223-230), batch of 3 rows each."""
    for z1 in range(1, 65):
        for z2 in range(1, 65):
            a = orc.gen_u32(11, 0, z1 * 100 + z2, 3, z1, p)
            b = orc.gen_u32(11, 1, z1 * 100 + z2, 3, z2, p)
            want, _, _ = orc.conv_batch(a, b, p, orc.ENGINE_TFT)
            got = _conv(a, b, p, engine)
            assert np.array_equal(got, want), (z1, z2, engine)


@pytest.mark.parametrize("p", [257, P2])
def test_sweep_128x128(orc, p):
    """Engine sweep over every (z1, z2) in (1..128)^2 (reference
    tests/test_acceptance.py:85-108); both engines."""
    for z1 in range(1, 129):
        for z2 in range(1, 129):
            n = z1 + z2 - 1
            if (n - 1).bit_length() > orc.two_adicity(p):
                continue
            a = orc.gen_u32(12, 0, z1 * 1000 + z2, 2, z1, p)
            b = orc.gen_u32(12, 1, z1 * 1000 + z2, 2, z2, p)
            want, _, _ = orc.conv_batch(a, b, p)
            for eng in ("fft_pad", "tft"):
                assert np.array_equal(_conv(a, b, p, eng), want), (p, z1, z2, eng)


@pytest.mark.parametrize("L", [2**k for k in range(0, 14)])
@pytest.mark.parametrize("p", [P1, P2, P3])
def test_power_of_two_boundaries(orc, L, p):
    """Products exactly at and just past each power-of-two length, plus the
    all-(p-1) operands that maximise every intermediate."""
    for n in sorted({L, L + 1, max(1, L - 1)}):
        for z1 in sorted({1, (n + 1) // 2, n}):
            z2 = n + 1 - z1
            if z2 < 1 or (n - 1).bit_length() > 13:
                continue
            a = orc.gen_u32(13, 0, n * 7 + z1, 4, z1, p)
            b = orc.gen_u32(13, 1, n * 7 + z1, 4, z2, p)
            a[0, :] = p - 1
            b[0, :] = p - 1
            b[1, :] = 0
            want, _, _ = orc.conv_batch(a, b, p)
            for eng in ("fft_pad", "tft"):
                assert np.array_equal(_conv(a, b, p, eng), want), (p, n, z1, eng)


@pytest.mark.parametrize("K", list(range(4, 14)))
@pytest.mark.parametrize("p", [P1, P3])
def test_fused_and_latency_paths_every_size(orc, K, p):
    """The fused kernel at every size with batches of 1, 40 and 300 (one CTA
    per product, a partial wave, more products than resident CTAs on the
    smaller sizes) -- same rows, bit-exact vs the oracle, at n = L and n just
    past L/2 (truncated transform), all-(p-1) rows."""
    L = 1 << K
    for n in (L, L // 2 + 1):
        z1 = (n + 1) // 3 + 1
        z2 = n + 1 - z1
        a = orc.gen_u32(14, 0, K * 10 + (n == L), 300, z1, p)
        b = orc.gen_u32(14, 1, K * 10 + (n == L), 300, z2, p)
        a[0, :] = p - 1
        b[0, :] = p - 1
        want, _, _ = orc.conv_batch(a, b, p, 1, threads=8)
        for eng in ("fft_pad", "tft"):
            for B in (1, 40, 300):
                got = _conv(a[:B], b[:B], p, eng)
                assert np.array_equal(got, want[:B]), (K, n, eng, B)


def test_cfg1_single_product(golden_configs):
    for cfg in golden_configs["configs"]:
        if cfg["cfg"] != 1:
            continue
        p = cfg["p"]
        a = gen_device(cfg["seed"], 0, 0, 1, cfg["z1"], p)
        b = gen_device(cfg["seed"], 1, 0, 1, cfg["z2"], p)
        for eng in ("fft_pad", "tft"):
            c = to_u32_np(mc.conv_batch(a, b, p, engine=eng))
            assert sha_row(c[0]) == cfg["rows"][0]["sha256"], eng


def test_cfg2_tft_batch(golden_configs, orc):
    cfg = next(c for c in golden_configs["configs"] if c["cfg"] == 2 and c["engine"] == "tft")
    p, z1, z2, B = cfg["p"], cfg["z1"], cfg["z2"], 4096
    a = gen_device(cfg["seed"], 0, 0, B, z1, p)
    b = gen_device(cfg["seed"], 1, 0, B, z2, p)
    c = mc.conv_batch(a, b, p, engine="tft")
    cn = to_u32_np(c)
    for rec in cfg["rows"]:
        assert sha_row(cn[rec["row"]]) == rec["sha256"], rec["row"]
    rng = np.random.default_rng(2)
    rows = sorted({0, B - 1, *(rng.integers(0, B, 24).tolist()), *range(0, B, 512),
                   *range(511, B, 512)})
    an, bn = to_u32_np(a), to_u32_np(b)
    want, _, _ = orc.conv_batch(an[rows], bn[rows], p, orc.ENGINE_TFT, threads=8)
    assert np.array_equal(cn[rows], want)
    eval_check(a, b, c, p)
    # the fft_pad engine on the same batch agrees bit for bit
    assert torch.equal(mc.conv_batch(a, b, p, engine="fft_pad"), c)


def test_cfg3_fft_pad_batch(golden_configs, orc):
    cfg = next(c for c in golden_configs["configs"] if c["cfg"] == 3)
    p, z1, z2, B = cfg["p"], cfg["z1"], cfg["z2"], 65536
    a = gen_device(cfg["seed"], 0, 0, B, z1, p)
    b = gen_device(cfg["seed"], 1, 0, B, z2, p)
    c = mc.conv_batch(a, b, p, engine="fft_pad")
    for rec in cfg["rows"]:
        assert sha_row(to_u32_np(c[rec["row"]])) == rec["sha256"], rec["row"]
    rng = np.random.default_rng(3)
    rows = sorted({0, B - 1, *(rng.integers(0, B, 32).tolist()), *range(0, B, 8192),
                   *range(8191, B, 8192)})
    idx = torch.tensor(rows, device="cuda")
    want, _, _ = orc.conv_batch(to_u32_np(a[idx]), to_u32_np(b[idx]), p, threads=8)
    assert np.array_equal(to_u32_np(c[idx]), want)
    eval_check(a, b, c, p)


def test_strided_rows_and_host_buffers(orc):
    p = P3
    a = gen_device(21, 0, 0, 5, 300, p, ld=512)
    b = gen_device(21, 1, 0, 5, 200, p, ld=256)
    want, _, _ = orc.conv_batch(to_u32_np(a), to_u32_np(b), p)
    assert np.array_equal(to_u32_np(mc.conv_batch(a, b, p)), want)
    ah, bh = a.cpu().pin_memory(), b.cpu().pin_memory()
    got = mc.conv_batch(ah, bh, p, engine="fft_pad")
    assert got.device.type == "cpu"
    assert np.array_equal(got.numpy().view(np.uint32), want)


@pytest.mark.parametrize("engine", ["fft_pad", "tft"])
def test_host_buffers_zero_copy_and_pipeline(orc, engine):
    """Host tensors: page-locked rows (zero copy: the kernel reads and writes
    host memory directly, strided rows included) and pageable rows (chunked
    copy pipeline) give the same bit-exact products."""
    p = P2
    B, z1, z2 = 700, 1500, 2100
    a = orc.gen_u32(22, 0, 0, B, z1, p)
    b = orc.gen_u32(22, 1, 0, B, z2, p)
    a[3, :] = p - 1
    b[3, :] = p - 1
    want, _, _ = orc.conv_batch(a, b, p, 1 if engine == "tft" else 0, threads=8)
    at = torch.from_numpy(a.view(np.int32))
    bt = torch.from_numpy(b.view(np.int32))
    # pinned, contiguous; output allocated by the call
    got = mc.conv_batch(at.pin_memory(), bt.pin_memory(), p, engine=engine)
    assert got.device.type == "cpu"
    assert np.array_equal(got.numpy().view(np.uint32), want)
    # pinned, strided rows in and out
    ap = torch.zeros((B, z1 + 37), dtype=torch.int32).pin_memory()
    bp = torch.zeros((B, z2 + 5), dtype=torch.int32).pin_memory()
    ap[:, :z1] = at
    bp[:, :z2] = bt
    cp = torch.full((B, z1 + z2 + 11), -1, dtype=torch.int32).pin_memory()
    out = cp[:, : z1 + z2 - 1]
    mc.conv_batch(ap[:, :z1], bp[:, :z2], p, engine=engine, out=out)
    assert np.array_equal(out.numpy().view(np.uint32), want)
    assert (cp[:, z1 + z2 - 1:] == -1).all()  # nothing written past n
    # pageable: the chunked copy pipeline
    got = mc.conv_batch(at.clone(), bt.clone(), p, engine=engine)
    assert np.array_equal(got.numpy().view(np.uint32), want)


@pytest.mark.parametrize("engine", ["fft_pad", "tft"])
def test_host_streamed_inputs(orc, monkeypatch, engine):
    """Streamed-input host mode (operand chunks H2D on a copy stream with
    per-chunk ready flags, one persistent kernel writing the page-locked
    output), forced at a small size; strided host rows included."""
    monkeypatch.setenv("MC_STREAM_IN_MIN_MB", "0")
    p = P3
    B, z1, z2 = 1100, 1499, 2102  # rows not a multiple of 4 words
    a = orc.gen_u32(24, 0, 0, B, z1, p)
    b = orc.gen_u32(24, 1, 0, B, z2, p)
    a[-1, :] = p - 1
    b[-1, :] = p - 1
    want = orc.conv_batch(a, b, p, 1 if engine == "tft" else 0, threads=8)[0]
    at = torch.from_numpy(a.view(np.int32)).pin_memory()
    bt = torch.from_numpy(b.view(np.int32)).pin_memory()
    got = mc.conv_batch(at, bt, p, engine=engine)
    assert np.array_equal(got.numpy().view(np.uint32), want)
    ap = torch.zeros((B, z1 + 9), dtype=torch.int32).pin_memory()
    ap[:, :z1] = at
    got = mc.conv_batch(ap[:, :z1], bt, p, engine=engine)
    assert np.array_equal(got.numpy().view(np.uint32), want)


@pytest.mark.parametrize("mode", ["zc", "ce", "in", "pipe"])
def test_host_modes_forced(orc, monkeypatch, mode):
    """Every host mode (zero copy, copy engines both ways, streamed inputs,
    chunked pipeline) forced
    on the same batch: bit-exact products, strided rows in and out, nothing
    written past n, staging reused across calls."""
    monkeypatch.setenv("MC_HOST_MODE", mode)
    p = P3
    B, z1, z2 = 1000, 1499, 2102
    n = z1 + z2 - 1
    a = orc.gen_u32(25, 0, 0, B, z1, p)
    b = orc.gen_u32(25, 1, 0, B, z2, p)
    a[0, :] = p - 1
    b[0, :] = p - 1
    want = orc.conv_batch(a, b, p, 1, threads=8)[0]
    at = torch.from_numpy(a.view(np.int32)).pin_memory()
    bt = torch.from_numpy(b.view(np.int32)).pin_memory()
    got = mc.conv_batch(at, bt, p, engine="tft")
    assert np.array_equal(got.numpy().view(np.uint32), want), mode
    cp = torch.full((B, n + 3), -1, dtype=torch.int32).pin_memory()
    ap = torch.zeros((B, z1 + 9), dtype=torch.int32).pin_memory()
    ap[:, :z1] = at
    for rep in range(2):  # reused staging buffers and counters
        mc.conv_batch(ap[:, :z1], bt, p, engine="tft", out=cp[:, :n])
        assert np.array_equal(cp[:, :n].numpy().view(np.uint32), want), (mode, rep)
        assert (cp[:, n:] == -1).all()


@pytest.mark.parametrize("mode", ["", "ce"])
def test_host_async_calls_on_two_streams(orc, monkeypatch, mode):
    """Two asynchronous host-buffer calls on different caller streams, issued
    back to back: the second must not overwrite the first's staging."""
    from paper_1609_01010_b200 import _native
    monkeypatch.setenv("MC_HOST_MODE", mode)
    p = P3
    B, z1, z2 = 600, 1500, 2100
    n = z1 + z2 - 1
    outs, wants = [], []
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    keep = []
    for k, st in enumerate(streams):
        a = orc.gen_u32(23 + k, 0, 0, B, z1, p)
        b = orc.gen_u32(23 + k, 1, 0, B, z2, p)
        wants.append(orc.conv_batch(a, b, p, 1, threads=8)[0])
        ah = torch.from_numpy(a.view(np.int32)).pin_memory()
        bh = torch.from_numpy(b.view(np.int32)).pin_memory()
        ch = torch.empty((B, n), dtype=torch.int32).pin_memory()
        keep += [ah, bh]
        outs.append(ch)
        _native.check(_native.lib().mc_conv_host_async(
            1, ah.data_ptr(), z1, z1, bh.data_ptr(), z2, z2, ch.data_ptr(), n, B, p, 0,
            st.cuda_stream))
    for st in streams:
        st.synchronize()
    for ch, want in zip(outs, wants):
        assert np.array_equal(ch.numpy().view(np.uint32), want)


def test_list_api_poly_mul(golden_small):
    for c in golden_small["poly_mul"]:
        fp = mc.FourierPrime.from_modulus(c["p"])
        cnt = mc.OpCounters()
        r = mc.poly_mul(mc.DensePoly(fp, tuple(c["u"])), mc.DensePoly(fp, tuple(c["v"])),
                        mc.ConvRequest(fp, engine=c["engine"], counters=cnt))
        assert list(r.coeffs) == c["out"]
        assert [cnt.butterflies, cnt.pointwise_muls] == c["counters"]


def test_concurrent_host_threads(orc):
    """Engines are reentrant (reference SPEC: pure, per-call counters): eight
    host threads multiplying at once on one device, list and tensor APIs,
    three fields (tables built concurrently), results bit-exact."""
    import threading

    results, errors = {}, []

    def work(k):
        try:
            p = (P1, P2, P3)[k % 3]
            fp = mc.FourierPrime.from_modulus(p)
            a = orc.gen_u32(80 + k, 0, 0, 6, 700 + 37 * k, p)
            b = orc.gen_u32(80 + k, 1, 0, 6, 500 + 11 * k, p)
            want = orc.conv_batch(a, b, p, 1)[0]
            got = mc.conv_batch(torch.from_numpy(a.view(np.int32)).cuda(),
                                torch.from_numpy(b.view(np.int32)).cuda(), p, engine="tft")
            torch.cuda.synchronize()
            cnt = mc.OpCounters()
            r = mc.poly_mul(mc.DensePoly(fp, tuple(a[0].tolist())), mc.DensePoly(fp, tuple(b[0].tolist())),
                            mc.ConvRequest(fp, engine="fft_pad", counters=cnt))
            results[k] = (np.array_equal(got.cpu().numpy().view(np.uint32), want),
                          list(r.coeffs) == want[0][:len(r.coeffs)].tolist())
        except Exception as exc:  # noqa: BLE001
            errors.append(repr(exc))

    ts = [threading.Thread(target=work, args=(k,)) for k in range(8)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    assert all(all(v) for v in results.values()) and len(results) == 8
