"""sm_100a kernels against the CPU oracle, bit for bit (-m gpu).

Tolerance: none. P, m, v and the 16-bit working params are compared as raw
bits; overflow and non-finite counts exactly. (north_star allows 1e-6 relative
on P/m/v and 1 ulp on 16-bit params; the kernel meets the stronger bar.)"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _dev(torch, a, dev):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def _u16(torch, a, dev):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).to(dev)


def _np16(t):
    return t.cpu().numpy().view(np.uint16)


def run_fused(tf, torch, dev, p, m, v, g16, t, gk=0, ok=0, wd=0.0, contiguous=False):
    n = p.size
    counters = torch.zeros(2, dtype=torch.int64, device=dev)
    p16 = torch.zeros(n, dtype=torch.int16, device=dev)
    hy = tf.AdamHyper(weight_decay=wd)
    if contiguous:
        st = _dev(torch, np.concatenate([p, m, v]), dev)
        g = _u16(torch, g16, dev)
        import ctypes as C
        from paper_2509_02480_b200 import _lib
        h = hy.c()
        _lib.call("tfg_adam_fused_contiguous", st.data_ptr(), n, g.data_ptr(), gk, p16.data_ptr(), ok, C.byref(h), t,
                  counters.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        s = st.cpu().numpy()
        return s[:n], s[n:2 * n], s[2 * n:], _np16(p16), counters.cpu().numpy()
    P, Mm, V, G = _dev(torch, p, dev), _dev(torch, m, dev), _dev(torch, v, dev), _u16(torch, g16, dev)
    tf.adam_fused(P, Mm, V, G, p16, t, hy, gk, ok, counters=counters)
    torch.cuda.synchronize()
    return P.cpu().numpy(), Mm.cpu().numpy(), V.cpu().numpy(), _np16(p16), counters.cpu().numpy()


def assert_bits(a, b, what):
    a32, b32 = np.asarray(a).view(np.uint32), np.asarray(b).view(np.uint32)
    bad = np.flatnonzero(a32 != b32)
    assert bad.size == 0, f"{what}: {bad.size} mismatches, first at {bad[:5]}: {a[bad[:3]]} vs {b[bad[:3]]}"


def test_contiguous_state_ten_steps_at_p_mod_4_eq_2(tf, cuda, golden):
    """The contiguous P||m||v kernel (m, v not 16-byte aligned at P % 4 = 2)
    for t = 1..10 with AdamW, against the reference's widen -> adam_step ->
    downscale chain (golden digests after every step, make_golden.py)."""
    import hashlib

    import torch
    n = 2_796_202
    st = _dev(torch, np.concatenate([oracle.synthetic_params(n, 42, 3), np.zeros(2 * n, np.float32)]), cuda)
    import ctypes as C
    from paper_2509_02480_b200 import _lib
    h = tf.AdamHyper(weight_decay=0.01).c()
    p16 = torch.zeros(n, dtype=torch.int16, device=cuda)
    counters = torch.zeros(2, dtype=torch.int64, device=cuda)
    for t in range(1, 11):
        g = _u16(torch, oracle.synthetic_grads(n, 42, 3, t - 1), cuda)
        _lib.call("tfg_adam_fused_contiguous", st.data_ptr(), n, g.data_ptr(), 0, p16.data_ptr(), 0, C.byref(h), t,
                  counters.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        s = st.cpu().numpy()
        assert hashlib.sha256(s.tobytes()).hexdigest() == golden["contig10_digest"][t - 1], f"t={t}"
        assert hashlib.sha256(_np16(p16).tobytes()).hexdigest() == golden["contig10_p16_digest"][t - 1], f"t={t}"
    assert_bits(s[::9973], golden["contig10_sample"], "sample")
    assert counters.cpu().tolist() == [0, 0]


def test_golden_vectors(tf, cuda, golden):
    import torch
    for k in range(int(golden["adam_cases"][0])):
        n, t, wd, over = golden[f"adam{k}_meta"]
        for contiguous in (False, True):
            p, m, v, p16, cnt = run_fused(tf, torch, cuda, golden[f"adam{k}_p"], golden[f"adam{k}_m"],
                                          golden[f"adam{k}_v"], golden[f"adam{k}_g16"], int(t), wd=wd,
                                          contiguous=contiguous)
            assert_bits(p, golden[f"adam{k}_p_out"], f"case {k} P")
            assert_bits(m, golden[f"adam{k}_m_out"], f"case {k} m")
            assert_bits(v, golden[f"adam{k}_v_out"], f"case {k} v")
            assert np.array_equal(p16, golden[f"adam{k}_p16"])
            assert cnt[0] == 0 and cnt[1] == int(over)


@pytest.mark.parametrize("n", [1, 3, 4, 5, 1023, 4096, 65537, 1 << 20, 3_000_001])
@pytest.mark.parametrize("gk,ok", [(0, 0), (0, 1), (1, 1), (1, 0)])
def test_random_sizes_and_dtypes(tf, cuda, n, gk, ok):
    import torch
    rng = np.random.default_rng(n * 7 + gk * 3 + ok)
    p = rng.uniform(-2, 2, n).astype(np.float32)
    m = (rng.uniform(-0.5, 0.5, n) * 0.1).astype(np.float32)
    v = rng.uniform(0, 0.01, n).astype(np.float32)
    g16 = oracle.synthetic_grads(n, 42, n % 97, 3, kind=gk)
    for t, wd in [(1, 0.0), (5, 0.01)]:
        want = oracle.adam_fused(p, m, v, g16, gk, ok, t, weight_decay=wd)
        got = run_fused(tf, torch, cuda, p, m, v, g16, t, gk, ok, wd)
        assert_bits(got[0], want[0], "P")
        assert_bits(got[1], want[1], "m")
        assert_bits(got[2], want[2], "v")
        assert np.array_equal(got[3], want[3])
        assert got[4][0] == 0 and got[4][1] == want[4]


def test_extreme_values(tf, cuda):
    """Subnormal moments, huge params overflowing 16-bit, zero grads, signed zeros."""
    import torch
    n = 8192
    rng = np.random.default_rng(1)
    p = np.concatenate([rng.uniform(-1e5, 1e5, n // 4), rng.uniform(-1e-30, 1e-30, n // 4),
                        np.full(n // 4, 65519.9, np.float32), np.array([0.0, -0.0] * (n // 8))]).astype(np.float32)
    m = np.concatenate([np.full(n // 2, 1e-40), rng.uniform(-1, 1, n // 2)]).astype(np.float32)
    v = np.concatenate([np.full(n // 2, 1e-44), rng.uniform(0, 1e-3, n // 2)]).astype(np.float32)
    g16 = np.concatenate([np.zeros(n // 4, np.uint16), np.full(n // 4, 0x8000, np.uint16),
                          oracle.f32_to_f16(rng.uniform(-60000, 60000, n // 2).astype(np.float32))])
    for t in (1, 2, 100, 10**6):
        for ok in (0, 1):
            want = oracle.adam_fused(p, m, v, g16, 0, ok, t, weight_decay=0.001)
            got = run_fused(tf, torch, cuda, p, m, v, g16, t, 0, ok, 0.001)
            for i in range(3):
                assert_bits(got[i], want[i], f"t={t} slot {i}")
            assert np.array_equal(got[3], want[3]) and got[4][1] == want[4]
            if ok == 0:
                assert want[4] > 0  # the fixture does exercise the f16 overflow counter


def test_nonfinite_gradients_are_counted_and_step_rejected(tf, cuda):
    import torch
    for n in (5000, 1000):  # the staged kernel (whole tiles) and the register kernel
        g16 = oracle.synthetic_grads(n, 1, 0, 0)
        g16[17] = 0x7C00
        g16[500] = 0x7E01
        g16[n - 1] = 0xFC00
        p = np.ones(n, np.float32)
        _, _, _, _, cnt = run_fused(tf, torch, cuda, p, p * 0, p * 0, g16, 1)
        assert cnt[0] == 3, n
    # reference semantics (optimizer.hpp:123-127): reject before mutating
    P = torch.ones(n, device=cuda)
    Mm, V = torch.zeros(n, device=cuda), torch.zeros(n, device=cuda)
    G = _u16(torch, g16, cuda)
    p16 = torch.zeros(n, dtype=torch.int16, device=cuda)
    with pytest.raises(tf.GradientOverflowError):
        tf.adam_step(P, Mm, V, G, p16, 1)
    assert bool((P == 1).all()) and bool((Mm == 0).all())
    with pytest.raises(tf.Error):
        tf.adam_step(P, Mm, V, G, p16, 0)  # t >= 1
    with pytest.raises(tf.ConfigError):
        tf.adam_step(P, Mm, V, G, p16, 1, tf.AdamHyper(beta1=1.0))


@pytest.mark.parametrize("gk,ok", [(0, 0), (1, 1)])
def test_gated_launch(tf, cuda, gk, ok):
    """A gated launch takes the gate as the whole-phase non-finite count: gate 0
    updates bit-exactly and counts overflows but not non-finite gradients
    (counters[0] stays 0); a nonzero gate writes nothing."""
    import torch
    n = 100_003
    rng = np.random.default_rng(3)
    p = rng.uniform(-7e4, 7e4, n).astype(np.float32)
    m = (rng.uniform(-0.5, 0.5, n) * 0.1).astype(np.float32)
    v = rng.uniform(0, 0.01, n).astype(np.float32)
    g16 = oracle.synthetic_grads(n, 42, 5, 2, kind=gk)
    want = oracle.adam_fused(p, m, v, g16, gk, ok, 3, weight_decay=0.0)
    assert want[4] > 0 or ok == 1  # f16 outputs overflow here, bf16 ones cannot
    P, Mm, V, G = _dev(torch, p, cuda), _dev(torch, m, cuda), _dev(torch, v, cuda), _u16(torch, g16, cuda)
    p16 = torch.zeros(n, dtype=torch.int16, device=cuda)
    counters = torch.zeros(2, dtype=torch.int64, device=cuda)
    gate = torch.ones(1, dtype=torch.int64, device=cuda)
    tf.adam_fused(P, Mm, V, G, p16, 3, tf.AdamHyper(), gk, ok, counters=counters, gate=gate)
    torch.cuda.synchronize()
    assert_bits(P.cpu().numpy(), p, "P untouched")
    assert int(counters.abs().sum()) == 0 and int(p16.abs().sum()) == 0
    gate.zero_()
    tf.adam_fused(P, Mm, V, G, p16, 3, tf.AdamHyper(), gk, ok, counters=counters, gate=gate)
    torch.cuda.synchronize()
    for got, w, what in ((P, want[0], "P"), (Mm, want[1], "m"), (V, want[2], "v")):
        assert_bits(got.cpu().numpy(), w, what)
    assert np.array_equal(_np16(p16), want[3])
    c = counters.cpu().numpy()
    assert c[0] == 0 and c[1] == want[4]


def test_adam_step_returns_overflows(tf, cuda):
    import torch
    n = 100
    P = torch.full((n,), 70000.0, device=cuda)
    Mm, V = torch.zeros(n, device=cuda), torch.zeros(n, device=cuda)
    G = torch.zeros(n, dtype=torch.int16, device=cuda)
    p16 = torch.zeros(n, dtype=torch.int16, device=cuda)
    assert tf.adam_step(P, Mm, V, G, p16, 1) == n


def test_synthetic_generators_bitwise(tf, cuda, golden):
    import torch
    for sg, it, steps in [(0, 0, 1), (3, 5, 1), (11, 2, 3)]:
        out = torch.zeros(4097, dtype=torch.int16, device=cuda)
        for s in range(steps):
            tf.synthetic_grads(out, 42, sg, it, s, accumulate=s > 0)
        torch.cuda.synchronize()
        assert np.array_equal(_np16(out), golden[f"grads_{sg}_{it}_{steps}"])
    for kind in (0, 1):
        out = torch.zeros(100003, dtype=torch.int16, device=cuda)
        for s in range(2):
            tf.synthetic_grads(out, 9, 4, 1, s, accumulate=s > 0, dtype=kind)
        assert np.array_equal(_np16(out), oracle.synthetic_grads(100003, 9, 4, 1, 2, kind))
    p = torch.empty(4097, device=cuda)
    m, v = torch.ones(4097, device=cuda), torch.ones(4097, device=cuda)
    tf.synthetic_state(p, m, v, 42, 9)
    assert_bits(p.cpu().numpy(), golden["params_42_9"], "param init")
    assert bool((m == 0).all()) and bool((v == 0).all())


def test_narrow_widen_exhaustive_f32(tf, cuda):
    """1/16 of all 2^32 float bit patterns (stride 16, every exponent and
    sign, NaN payloads included) narrowed to f16 and bf16 on the GPU agree
    with the oracle bit for bit, and the overflow counters agree."""
    import torch
    chunk = 1 << 26
    out = torch.empty(chunk, dtype=torch.int16, device=cuda)
    over = torch.zeros(1, dtype=torch.int64, device=cuda)
    total_over = [0, 0]
    for kind in (0, 1):
        for q in range(4):  # stride-16 sample of each quarter of the 2^32 patterns (every exponent)
            base = q * (1 << 30) + (q * 5 + 3) % 16
            idx = torch.arange(chunk, dtype=torch.int64, device=cuda) * 16 + base
            bits = idx.to(torch.int32).view(torch.float32)
            tf.downscale16(bits, out, kind, over)
            want, o = oracle.narrow16(bits.cpu().numpy(), kind)
            assert np.array_equal(_np16(out), want), (kind, q)
            total_over[kind] += o
        assert int(over.item()) == total_over[kind]
        over.zero_()
    # widen: every 16-bit pattern
    h = torch.arange(65536, dtype=torch.int32, device=cuda).to(torch.int16)
    f = torch.empty(65536, device=cuda)
    nf = torch.zeros(1, dtype=torch.int64, device=cuda)
    for kind in (0, 1):
        tf.upscale16(h, f, kind, nf)
        want = oracle.widen16(np.arange(65536, dtype=np.uint16), kind)
        got = f.cpu().numpy()
        fin = ~np.isnan(want)
        assert_bits(got[fin], want[fin], "widen")
        assert np.isnan(got[~fin]).all()
    assert int(nf.item()) == 2048 + 256  # non-finite f16 + bf16 patterns


def test_constant_division_matches_div_rn(tf, cuda):
    """m/bc1 and v/bc2 through the hoisted-reciprocal quotient equal div.rn.f64
    for the bias corrections of several (beta, t), on generated numerators."""
    for beta in (0.9, 0.999, 0.5, 0.95, 0.0):
        for t in (1, 2, 3, 10, 1000, 10**6):
            bc = 1.0 - beta ** t
            mism, first = tf.selftest_div_const(bc, 2_000_000, seed=t)
            assert mism == 0, (beta, t, first)


@pytest.mark.parametrize("variant", [v for v in range(1, 72) if v != 67])  # 67: tile-interleaved layout
def test_kernel_variants_bitwise(tf, cuda, variant):
    import torch
    n = 1_000_003
    rng = np.random.default_rng(variant)
    p = rng.uniform(-2, 2, n).astype(np.float32)
    m = (rng.uniform(-0.5, 0.5, n) * 0.1).astype(np.float32)
    v = rng.uniform(0, 0.01, n).astype(np.float32)
    g16 = oracle.synthetic_grads(n, 42, variant, 1)
    want = oracle.adam_fused(p, m, v, g16, 0, 0, 4, weight_decay=0.01)
    P, Mm, V, G = _dev(torch, p, cuda), _dev(torch, m, cuda), _dev(torch, v, cuda), _u16(torch, g16, cuda)
    p16 = torch.zeros(n, dtype=torch.int16, device=cuda)
    tf.adam_fused_variant(variant, P, Mm, V, G, p16, 4, tf.AdamHyper(weight_decay=0.01))
    torch.cuda.synchronize()
    assert_bits(P.cpu().numpy(), want[0], "P")
    assert_bits(Mm.cpu().numpy(), want[1], "m")
    assert_bits(V.cpu().numpy(), want[2], "v")
    assert np.array_equal(_np16(p16), want[3])


def test_fast_step_error_bound_and_bits(tf, cuda):
    """The second verified fast path (tuning variants 44-46): its approximate
    step stays within 2^-30 relative of the exact chain's (the tolerance its
    acceptance test assumes) over 2^26 random (m, v, t) spanning 40-80
    binades, and the P/m/v bits it produces equal the shipped kernel's."""
    import ctypes as C

    from paper_2509_02480_b200 import _lib
    worst, mism = C.c_double(), C.c_uint64()
    _lib.call_tuning("tfg_selftest_fast_step", 1 << 26, 2026, C.byref(worst), C.byref(mism))
    assert mism.value == 0
    assert worst.value < 2.0 ** -30, worst.value


def test_in_range_sqrt_and_division_are_correctly_rounded(tf, cuda):
    """Variant 47's sqrt / division without the special-operand checks equal
    __dsqrt_rn / __ddiv_rn bit for bit on 2^28 random operand pairs over the
    exponent ranges the Adam chain keeps them in (fast_rn_domain)."""
    import ctypes as C

    from paper_2509_02480_b200 import _lib
    bad = C.c_uint64()
    for seed in (1, 2, 3, 4):
        _lib.call_tuning("tfg_selftest_fast_rn", 1 << 26, seed, C.byref(bad))
        assert bad.value == 0, seed


@pytest.mark.parametrize("nsrc", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("kind", [0, 1])
def test_fused_reduce_update_matches_oracle(tf, cuda, nsrc, kind):
    """tfg_adam_fused_multi: gradient = fp32 sum of n 16-bit sources in order,
    rounded once, then Adam — the reduce-scatter fused into the update."""
    import torch
    n = 300_001
    rng = np.random.default_rng(nsrc * 10 + kind)
    srcs = [oracle.synthetic_grads(n, 77, s, 2, kind=kind) for s in range(nsrc)]
    for s in srcs:  # negative zeros in every source sum to -0 (the sum starts at source 0)
        s[:64] = 0x8000
    acc = np.full(n, -0.0, np.float32)
    for s in srcs:
        acc = (acc + oracle.widen16(s, kind)).astype(np.float32)
    g16, _ = oracle.narrow16(acc, kind)
    p = rng.uniform(-1, 1, n).astype(np.float32)
    m = (rng.uniform(-0.5, 0.5, n) * 0.1).astype(np.float32)
    v = rng.uniform(0, 0.01, n).astype(np.float32)
    want = oracle.adam_fused(p, m, v, g16, kind, kind, 3, weight_decay=0.01)
    P, Mm, V = _dev(torch, p, cuda), _dev(torch, m, cuda), _dev(torch, v, cuda)
    G = [_u16(torch, s, cuda) for s in srcs]
    p16 = torch.zeros(n, dtype=torch.int16, device=cuda)
    counters = torch.zeros(2, dtype=torch.int64, device=cuda)
    tf.adam_fused_multi(P, Mm, V, G, p16, 3, tf.AdamHyper(weight_decay=0.01), kind, kind, counters)
    torch.cuda.synchronize()
    assert_bits(P.cpu().numpy(), want[0], "P")
    assert_bits(Mm.cpu().numpy(), want[1], "m")
    assert_bits(V.cpu().numpy(), want[2], "v")
    assert np.array_equal(_np16(p16), want[3])
    assert counters.cpu().tolist() == [0, want[4]]


@pytest.mark.parametrize("nsrc", [2, 4, 8])
@pytest.mark.parametrize("form", [0, 1])
def test_multi_source_forms_match_oracle(tf, cuda, nsrc, form):
    """Both n-source kernels (tuning hook: 0 = staged, 1 = register) against the
    oracle, f16, a partial tile at the end; non-finite sums are counted."""
    import torch
    n = 1 << 20 | 515
    rng = np.random.default_rng(nsrc * 7 + form)
    srcs = [oracle.synthetic_grads(n, 91, s, 1) for s in range(nsrc)]
    srcs[0][5] = 0x7C00  # one +Inf contribution: a non-finite sum
    acc = np.full(n, -0.0, np.float32)
    for s in srcs:
        acc = (acc + oracle.widen16(s, 0)).astype(np.float32)
    g16, _ = oracle.narrow16(acc, 0)
    g16[5] = 0  # the oracle rejects a non-finite step: compare every other element
    p = rng.uniform(-1, 1, n).astype(np.float32)
    m = (rng.uniform(-0.5, 0.5, n) * 0.1).astype(np.float32)
    v = rng.uniform(0, 0.01, n).astype(np.float32)
    want = oracle.adam_fused(p, m, v, g16, 0, 0, 2, weight_decay=0.0)
    P, Mm, V = _dev(torch, p, cuda), _dev(torch, m, cuda), _dev(torch, v, cuda)
    G = [_u16(torch, s, cuda) for s in srcs]
    p16 = torch.zeros(n, dtype=torch.int16, device=cuda)
    counters = torch.zeros(2, dtype=torch.int64, device=cuda)
    tf.adam_fused_multi_variant(form, P, Mm, V, G, p16, 2, tf.AdamHyper(), counters)
    torch.cuda.synchronize()
    keep = np.ones(n, bool)
    keep[5] = False
    for got, w, what in ((P, want[0], "P"), (Mm, want[1], "m"), (V, want[2], "v")):
        assert_bits(got.cpu().numpy()[keep], w[keep], what)
    assert np.array_equal(_np16(p16)[keep], want[3][keep])
    assert counters.cpu().tolist()[0] == 1


def test_fp32_gradient_kind(tf, cuda):
    """grad_dtype F32: the baseline flow's stored fp32 gradients."""
    import torch
    import ctypes as C
    from paper_2509_02480_b200 import _lib
    n = 100_003
    rng = np.random.default_rng(4)
    g = oracle.widen16(oracle.synthetic_grads(n, 5, 1, 1), 0).copy()
    p = rng.uniform(-1, 1, n).astype(np.float32)
    m, v = np.zeros(n, np.float32), np.zeros(n, np.float32)
    wp, wm, wv = p.copy(), m.copy(), v.copy()
    assert oracle.lib().orc_adam_step(wp, wm, wv, g, n, 1e-3, 0.9, 0.999, 1e-8, 0.0, 2) == 0
    P, Mm, V, Gd = (_dev(torch, x, cuda) for x in (p, m, v, g))
    p16 = torch.zeros(n, dtype=torch.int16, device=cuda)
    h = tf.AdamHyper().c()
    _lib.call("tfg_adam_fused", P.data_ptr(), Mm.data_ptr(), V.data_ptr(), Gd.data_ptr(), tf.F32, p16.data_ptr(),
              0, n, C.byref(h), 2, None, None)
    torch.cuda.synchronize()
    assert_bits(P.cpu().numpy(), wp, "P")
    assert_bits(Mm.cpu().numpy(), wm, "m")
    assert_bits(V.cpu().numpy(), wv, "v")
    assert np.array_equal(_np16(p16), oracle.f32_to_f16(wp))


def _near_midpoint_inputs(count=40, seed=11, t=3, tol_bits=96):
    """Elements whose exact p_new = RN64(p - D) lies within `tol_bits` double
    ulps of a binary32 rounding midpoint: the cases the verified fast path
    must hand to the exact chain. Found by a vectorised search in float64
    (numpy rounds every op, no contraction: the reference chain)."""
    rng = np.random.default_rng(seed)
    lr, b1, b2, eps = 1e-3, 0.9, 0.999, 1e-8
    bc1, bc2 = 1 - b1 ** t, 1 - b2 ** t
    found = [np.empty(0, np.float32)] * 4
    while found[0].size < count:
        n = 4_000_000
        p = rng.uniform(-2, 2, n).astype(np.float32)
        m = (rng.uniform(-0.5, 0.5, n) * 0.1).astype(np.float32)
        v = rng.uniform(0, 0.01, n).astype(np.float32)
        g16 = oracle.f32_to_f16(rng.uniform(-0.25, 0.25, n).astype(np.float32))
        g = oracle.widen16(g16, 0).astype(np.float64)
        m64 = b1 * m.astype(np.float64) + (1 - b1) * g
        v64 = b2 * v.astype(np.float64) + ((1 - b2) * g) * g
        pn = p.astype(np.float64) - (lr * (m64 / bc1)) / (np.sqrt(v64 / bc2) + eps)
        low = pn.view(np.uint64) & np.uint64((1 << 29) - 1)
        dist = np.abs(low.astype(np.int64) - (1 << 28))
        sel = dist <= tol_bits
        found = [np.concatenate([f, x[sel]]) for f, x in zip(found, (p, m, v, g16.astype(np.float32)))]
    return found[0], found[1], found[2], found[3].astype(np.uint16), t


@pytest.mark.parametrize("variant", [0, 18, 19])
def test_fast_path_fallback_on_midpoint_cases(tf, cuda, variant):
    import torch
    p, m, v, g16, t = _near_midpoint_inputs()
    rng = np.random.default_rng(5)
    n_fill = 100_000
    p = np.concatenate([p, rng.uniform(-2, 2, n_fill).astype(np.float32)])
    m = np.concatenate([m, (rng.uniform(-0.5, 0.5, n_fill) * 0.1).astype(np.float32)])
    v = np.concatenate([v, rng.uniform(0, 0.01, n_fill).astype(np.float32)])
    g16 = np.concatenate([g16, oracle.synthetic_grads(n_fill, 3, 3, 3)])
    want = oracle.adam_fused(p, m, v, g16, 0, 0, t)
    P, Mm, V, G = _dev(torch, p, cuda), _dev(torch, m, cuda), _dev(torch, v, cuda), _u16(torch, g16, cuda)
    p16 = torch.zeros(p.size, dtype=torch.int16, device=cuda)
    tf.adam_fused_variant(variant, P, Mm, V, G, p16, t, tf.AdamHyper())
    torch.cuda.synchronize()
    assert_bits(P.cpu().numpy(), want[0], "P")
    assert_bits(Mm.cpu().numpy(), want[1], "m")
    assert_bits(V.cpu().numpy(), want[2], "v")
    assert np.array_equal(_np16(p16), want[3])


def test_one_billion_param_subgroup_is_chunk_invariant(tf, cuda):
    """SURVEY C5 upper end (1B params per subgroup, 12 GB of state): one launch
    over the whole subgroup equals ten launches over 100M-param slices, bit
    for bit (element-wise op; exercises 64-bit indexing past 2^32 bytes), and
    the counters agree."""
    import torch
    n = 1_000_000_000
    st = torch.empty(3 * n, dtype=torch.float32, device=cuda)
    g = torch.empty(n, dtype=torch.int16, device=cuda)
    tf.synthetic_state(st[:n], st[n:2 * n], st[2 * n:], 7, 3)
    tf.synthetic_grads(g, 7, 3, 0)
    ref = st.clone()
    idx = np.random.default_rng(1).integers(0, n, 4096)
    ti = torch.from_numpy(idx).to(cuda)
    p0 = st[ti].cpu().numpy()
    m0 = st[n + ti].cpu().numpy()
    v0 = st[2 * n + ti].cpu().numpy()
    g0 = g[ti].cpu().numpy().view(np.uint16)
    p16a = torch.empty(n, dtype=torch.int16, device=cuda)
    p16b = torch.empty(n, dtype=torch.int16, device=cuda)
    ca = torch.zeros(2, dtype=torch.int64, device=cuda)
    cb = torch.zeros(2, dtype=torch.int64, device=cuda)
    hy = tf.AdamHyper(weight_decay=0.01)
    tf.adam_fused(st[:n], st[n:2 * n], st[2 * n:], g, p16a, 5, hy, counters=ca)
    c = 100_000_000
    for k in range(0, n, c):
        tf.adam_fused(ref[k:k + c], ref[n + k:n + k + c], ref[2 * n + k:2 * n + k + c], g[k:k + c], p16b[k:k + c],
                      5, hy, counters=cb)
    torch.cuda.synchronize()
    assert torch.equal(st.view(torch.int32), ref.view(torch.int32))
    assert torch.equal(p16a, p16b)
    assert ca.tolist() == cb.tolist()
    # and a sample of elements, far into the buffer, against the CPU oracle
    want = oracle.adam_fused(p0, m0, v0, g0, 0, 0, 5, weight_decay=0.01)
    assert np.array_equal(st[ti].cpu().numpy().view(np.uint32), want[0].view(np.uint32))
    assert np.array_equal(st[n + ti].cpu().numpy().view(np.uint32), want[1].view(np.uint32))
    assert np.array_equal(st[2 * n + ti].cpu().numpy().view(np.uint32), want[2].view(np.uint32))
    assert np.array_equal(p16a[ti].cpu().numpy().view(np.uint16), want[3])


# Tile edges of the shipped staged shape (2048-param tiles, 2 CTAs x 512 threads per SM on 148 SMs):
# one tile, one tile +-1, a partial quad, one full wave of CTAs plus a 577-param tail.
@pytest.mark.gpu
@pytest.mark.parametrize("n", [2048, 2049, 4095, 4097, 2048 * 296 + 577, 2048 * 296 * 3 + 2, 1_000_001])
def test_staged_tile_edges_and_canaries(tf, cuda, n):
    """Bits equal the oracle at the tile edges, and nothing outside [0, n) is written: every stream sits
    between 16-byte-aligned canary regions (the kernel's own bounds, checked without a sanitizer)."""
    import torch
    pad = 4096
    rng = np.random.default_rng(n)
    p = rng.uniform(-2, 2, n).astype(np.float32)
    m = (rng.uniform(-0.5, 0.5, n) * 0.1).astype(np.float32)
    v = rng.uniform(0, 0.01, n).astype(np.float32)
    g16 = oracle.synthetic_grads(n, 7, n % 31, 2, kind=0)
    want = oracle.adam_fused(p, m, v, g16, 0, 0, 3, weight_decay=0.01)

    def framed(a, dtype, fill):
        buf = torch.full((pad + a.size + pad,), fill, dtype=dtype, device=cuda)
        buf[pad:pad + a.size] = torch.from_numpy(a.view(np.int16) if dtype == torch.int16 else a).to(cuda)
        return buf

    P, M, V = (framed(a, torch.float32, 1234.5) for a in (p, m, v))
    G = framed(g16, torch.int16, 0x3C00)
    P16 = torch.full((pad + n + pad,), 0x7E00, dtype=torch.int16, device=cuda)
    counters = torch.zeros(2, dtype=torch.int64, device=cuda)
    sl = slice(pad, pad + n)
    tf.adam_fused(P[sl], M[sl], V[sl], G[sl], P16[sl], 3, tf.AdamHyper(weight_decay=0.01), 0, 0, counters=counters)
    torch.cuda.synchronize()
    for name, buf, fill in (("P", P, 1234.5), ("m", M, 1234.5), ("v", V, 1234.5)):
        h = buf.cpu().numpy()
        assert np.all(h[:pad] == fill) and np.all(h[pad + n:] == fill), f"{name}: write outside [0, n)"
    h16 = P16.cpu().numpy()
    assert np.all(h16[:pad] == 0x7E00) and np.all(h16[pad + n:] == 0x7E00), "params16: write outside [0, n)"
    assert_bits(P[sl].cpu().numpy(), want[0], "P")
    assert_bits(M[sl].cpu().numpy(), want[1], "m")
    assert_bits(V[sl].cpu().numpy(), want[2], "v")
    assert np.array_equal(_np16(P16[sl]), want[3])
    assert counters.cpu().numpy()[1] == want[4]


@pytest.mark.gpu
@pytest.mark.parametrize("nsrc", [2, 8])
@pytest.mark.parametrize("n", [4097, 2048 * 296 + 577])
def test_multi_source_canaries(tf, cuda, nsrc, n):
    """The n-source reduce + update (8 sources: the staged form) writes nothing outside [0, n) and reads
    its sources only inside [0, n): a source's out-of-range neighbours are NaN, so a stray read of one
    would reach the non-finite counter or the bits."""
    import torch
    pad = 4096
    rng = np.random.default_rng(nsrc * 1000 + n)
    srcs = [oracle.synthetic_grads(n, 5, s, 2, kind=0) for s in range(nsrc)]
    acc = np.full(n, -0.0, np.float32)
    for s in srcs:
        acc = (acc + oracle.widen16(s, 0)).astype(np.float32)
    g16, _ = oracle.narrow16(acc, 0)
    p = rng.uniform(-1, 1, n).astype(np.float32)
    m = (rng.uniform(-0.5, 0.5, n) * 0.1).astype(np.float32)
    v = rng.uniform(0, 0.01, n).astype(np.float32)
    want = oracle.adam_fused(p, m, v, g16, 0, 0, 2, weight_decay=0.01)

    def framed(a, dtype, fill):
        buf = torch.full((pad + a.size + pad,), fill, dtype=dtype, device=cuda)
        buf[pad:pad + a.size] = torch.from_numpy(a.view(np.int16) if dtype == torch.int16 else a).to(cuda)
        return buf

    sl = slice(pad, pad + n)
    P, M, V = (framed(a, torch.float32, -77.25) for a in (p, m, v))
    G = [framed(s, torch.int16, 0x7E00) for s in srcs]  # f16 NaN around every source
    P16 = torch.full((pad + n + pad,), 0x1234, dtype=torch.int16, device=cuda)
    counters = torch.zeros(2, dtype=torch.int64, device=cuda)
    tf.adam_fused_multi(P[sl], M[sl], V[sl], [g[sl] for g in G], P16[sl], 2, tf.AdamHyper(weight_decay=0.01), 0, 0,
                        counters)
    torch.cuda.synchronize()
    for name, buf in (("P", P), ("m", M), ("v", V)):
        h = buf.cpu().numpy()
        assert np.all(h[:pad] == -77.25) and np.all(h[pad + n:] == -77.25), f"{name}: write outside [0, n)"
    h16 = P16.cpu().numpy()
    assert np.all(h16[:pad] == 0x1234) and np.all(h16[pad + n:] == 0x1234), "params16: write outside [0, n)"
    assert_bits(P[sl].cpu().numpy(), want[0], "P")
    assert_bits(M[sl].cpu().numpy(), want[1], "m")
    assert_bits(V[sl].cpu().numpy(), want[2], "v")
    assert np.array_equal(_np16(P16[sl]), want[3])
    assert counters.cpu().tolist() == [0, want[4]]
