"""Generates tests/golden/golden.npz from the UNMODIFIED reference headers
compiled in place (oracle/_ref/libtierflow_ref.so, built by `make -C oracle`
from /root/reference/proj/include). Re-run here (not on the GPU box, which has
no /root/reference):

    python tests/golden/make_golden.py

Every array below is a reference output on seeded inputs; the tests pin the
C restatement (oracle/liboracle.so) and, on the GPU, the CUDA path to them.
"""
from __future__ import annotations

import hashlib
import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402

OUT = Path(__file__).resolve().parent / "golden.npz"


def adam_inputs(n, seed):
    # Distributions of the reference's own optimizer tests (test_optimizer.cpp:31-42).
    rng = np.random.default_rng(seed)
    p = rng.uniform(-2.0, 2.0, n).astype(np.float32)
    m = (rng.uniform(-0.5, 0.5, n) * 0.1).astype(np.float32)
    v = rng.uniform(0.0, 0.01, n).astype(np.float32)
    return p, m, v


def main() -> None:
    R = oracle.ref()
    g = {}
    rng = np.random.default_rng(20250902)

    # f16 narrowing: the reference spot values (test_precision.cpp:68-96) + random floats.
    spots = np.array([1.0, -2.5, 65504.0, 1 + 2**-12, 1 + 2**-11, 1 + 3 * 2**-12, 65519.0, 65520.0, 70000.0,
                      -70000.0, 2**-24, 2**-25, 1.5 * 2**-25, 2**-26, -0.0, np.inf, -np.inf, np.nan], np.float32)
    rand = (rng.standard_normal(20000) * np.exp2(rng.integers(-28, 18, 20000))).astype(np.float32)
    x = np.concatenate([spots, rand])
    g["f16_x"] = x
    g["f16_bits"] = np.array([R.ref_f32_to_f16(float(v)) for v in x], np.uint16)

    # Adam cases: contiguous widen(g16) -> adam_step -> downscale.
    cases = [(4099, 1, 0.0), (4099, 2, 0.01), (1031, 7, 0.0), (1031, 1000, 0.1), (1, 1, 0.0)]
    for k, (n, t, wd) in enumerate(cases):
        p, m, v = adam_inputs(n, 100 + k)
        g16 = oracle.synthetic_grads(n, 42, k, t)  # finite binary16 gradients in [-0.25, 0.25)
        gf = np.empty(n, np.float32)
        fin = oracle.C.c_int()
        R.ref_upscale(g16, gf, n, oracle.C.byref(fin))
        po, mo, vo = p.copy(), m.copy(), v.copy()
        assert R.ref_adam_step(po, mo, vo, gf, n, 1e-3, 0.9, 0.999, 1e-8, wd, t, 2) == 0
        p16 = np.empty(n, np.uint16)
        over = oracle.C.c_uint64()
        R.ref_downscale(po, p16, n, oracle.C.byref(over))
        for name, arr in dict(p=p, m=m, v=v, g16=g16, p_out=po, m_out=mo, v_out=vo, p16=p16).items():
            g[f"adam{k}_{name}"] = arr
        g[f"adam{k}_meta"] = np.array([n, t, wd, over.value], np.float64)
    g["adam_cases"] = np.array([len(cases)])

    # Hand oracle of test_optimizer.cpp:55-72 (fp32 g = 0.1).
    p, m, v = np.array([1.0], np.float32), np.zeros(1, np.float32), np.zeros(1, np.float32)
    R.ref_adam_step(p, m, v, np.array([0.1], np.float32), 1, 1e-3, 0.9, 0.999, 1e-8, 0.0, 1, 1)
    g["hand_pmv"] = np.concatenate([p, m, v])

    # Synthetic generators (scheduler.hpp:85-110).
    for sg, it, steps in [(0, 0, 1), (3, 5, 1), (11, 2, 3)]:
        out = np.zeros(4097, np.uint16)
        R.ref_accumulated_grads(out, 4097, 42, sg, it, steps)
        g[f"grads_{sg}_{it}_{steps}"] = out
    prm = np.empty(4097, np.float32)
    R.ref_synthetic_params(prm, 4097, 42, 9)
    g["params_42_9"] = prm

    # Placement (Eq. 1) and destination plans.
    Ms, bws, counts = [], [], []
    for _ in range(300):
        N = int(rng.integers(1, 5))
        M = int(rng.integers(1, 65))
        bw = np.where(rng.random(N) < 0.05, 0.0, 10 ** rng.uniform(-1.5, 1.5, N))
        if not (bw > 0).any():
            bw[0] = 1.0
        c = np.zeros(N, np.int32)
        assert R.ref_assign_subgroups(M, bw, N, c) == 0
        Ms.append(M)
        bws.append(np.pad(bw, (0, 4 - N), constant_values=-1.0))
        counts.append(np.pad(c, (0, 4 - N), constant_values=-1))
    g["eq1_M"], g["eq1_bw"], g["eq1_counts"] = np.array(Ms), np.array(bws), np.array(counts)

    # Engine runs on throttled in-memory tiers with a pinned placement ratio.
    with tempfile.TemporaryDirectory() as locks:
        runs = {
            # cache hits {0,4,4,4} (test_scheduler.cpp:286-301), M=12, C=4
            "hits": dict(params=[20000] * 12, tiers=[(500e6, 500e6), (250e6, 250e6)], ratio=[2.0, 1.0],
                         pool_slots=7, cache_slots=-1, seed=21, iterations=4, accum=1, wd=0.0, skip=0),
            # ragged subgroups (P % 4 != 0), three tiers, accumulation, decay, C=2
            "ragged": dict(params=[3001, 3001, 3001, 3001, 3001, 1234], tiers=[(300e6, 300e6), (200e6, 200e6),
                                                                                (100e6, 100e6)],
                           ratio=[3.0, 2.0, 1.0], pool_slots=5, cache_slots=-1, seed=7, iterations=5, accum=2,
                           wd=0.01, skip=0),
            # a skipped iteration keeps the parity key (SURVEY.md §8a rule 2)
            "skip": dict(params=[5000] * 8, tiers=[(400e6, 400e6), (200e6, 200e6)], ratio=[1.0, 1.0],
                         pool_slots=6, cache_slots=2, seed=5, iterations=4, accum=1, wd=0.0, skip=0b10),
            # the north_star "after 10 steps" contract on the reference desk shape (configs/desk.json:
            # 24 x 2,796,202, P % 4 = 2): 12 iterations, iteration 5 skipped (11 applied), C = 4, AdamW
            "desk10": dict(params=[2_796_202] * 24, tiers=[(4000e6, 4000e6), (2000e6, 2000e6)], ratio=[2.0, 1.0],
                           pool_slots=7, cache_slots=-1, seed=42, iterations=12, accum=1, wd=0.01, skip=1 << 5),
            # the ZeRO-3 baseline flow: caching, skip-gradients, atomic R/W and multi-path all off
            "baseline": dict(params=[20000] * 6, tiers=[(300e6, 300e6), (150e6, 150e6)], ratio=None,
                             pool_slots=6, cache_slots=-1, seed=1234, iterations=3, accum=2, wd=0.0, skip=0,
                             mode="baseline"),
        }
        for name, c in runs.items():
            tiers = [dict(kind=2, read_bps=r, write_bps=w) for r, w in c["tiers"]]
            base = c.get("mode") == "baseline"
            res = oracle.run_ref_engine(c["params"], tiers, fixed_ratio=c["ratio"], pool_slots=c["pool_slots"],
                                        cache_slots=c["cache_slots"], seed=c["seed"], iterations=c["iterations"],
                                        accum_steps=c["accum"], weight_decay=c["wd"], skip_mask=c["skip"],
                                        lock_dir=locks, enable_caching=not base, multi_path=not base,
                                        atomic_rw=not base, skip_gradients=not base)
            # storage bytes per iteration: backward flushes, update-phase fetches
            bw_bytes, up_bytes, prev = [], [], 0
            for it in res["iters"]:
                ev = res["events"]
                bw_bytes.append(sum(b for k, _s, _t, b in ev[prev:it["trace_begin"]] if k == oracle.EV_FLUSH_END))
                up_bytes.append(sum(b for k, _s, _t, b in ev[it["trace_begin"]:it["trace_end"]]
                                    if k == oracle.EV_PREFETCH_END))
                prev = it["trace_end"]
            g[f"run_{name}_backward_bytes"] = np.array(bw_bytes, np.int64)
            g[f"run_{name}_fetch_bytes"] = np.array(up_bytes, np.int64)
            g[f"run_{name}_config"] = np.array(
                [len(c["params"]), len(c["tiers"]), c["pool_slots"], c["cache_slots"], c["seed"], c["iterations"],
                 c["accum"], c["skip"]], np.int64)
            g[f"run_{name}_params"] = np.array(c["params"], np.int64)
            g[f"run_{name}_ratio"] = np.array(c["ratio"] if c["ratio"] else [], np.float64)
            g[f"run_{name}_wd"] = np.array([c["wd"]])
            g[f"run_{name}_hits"] = np.array([it["cache_hits"] for it in res["iters"]], np.int64)
            g[f"run_{name}_retained"] = np.array([it["retained"] for it in res["iters"]], np.int64)
            g[f"run_{name}_alloc"] = np.array([it["flush_allocation"] for it in res["iters"]], np.int64)
            g[f"run_{name}_overflows"] = np.array([it["overflows"] for it in res["iters"]], np.int64)
            nt = len(c["tiers"])
            seqs = []
            for it in res["iters"]:
                s = oracle.phase_sequences(res["events"], it["trace_begin"], it["trace_end"], nt)
                seqs.append(repr(s))
            g[f"run_{name}_seqs"] = np.array(seqs)
            if name in ("hits", "baseline", "desk10"):  # large: keep a digest per subgroup
                g[f"run_{name}_digest"] = np.array([hashlib.sha256(x.tobytes()).hexdigest() for x in res["states"]])
            else:
                g[f"run_{name}_states"] = np.concatenate(res["states"])
    # The contiguous P||m||v kernel (StateView::from_contiguous, optimizer.hpp:82-86) for t = 1..10 at
    # the desk shape's P = 2,796,202 (P % 4 = 2: m and v are not 16-byte aligned): widen the fp16
    # SyntheticGradSource gradient, adam_step with AdamW, downscale; digests after every step.
    n = 2_796_202
    state = np.concatenate([oracle.synthetic_params(n, 42, 3), np.zeros(2 * n, np.float32)])
    dig, dig16 = [], []
    for t in range(1, 11):
        g16 = oracle.synthetic_grads(n, 42, 3, t - 1)
        gf = np.empty(n, np.float32)
        fin = oracle.C.c_int()
        R.ref_upscale(g16, gf, n, oracle.C.byref(fin))
        p, m, v = state[:n], state[n:2 * n], state[2 * n:]
        assert R.ref_adam_step(p, m, v, gf, n, 1e-3, 0.9, 0.999, 1e-8, 0.01, t, 4) == 0
        p16 = np.empty(n, np.uint16)
        over = oracle.C.c_uint64()
        R.ref_downscale(p, p16, n, oracle.C.byref(over))
        dig.append(hashlib.sha256(state.tobytes()).hexdigest())
        dig16.append(hashlib.sha256(p16.tobytes()).hexdigest())
    g["contig10_digest"] = np.array(dig)
    g["contig10_p16_digest"] = np.array(dig16)
    g["contig10_sample"] = state[::9973].copy()  # a readable sample of the final state

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(g)} arrays)")


if __name__ == "__main__":
    main()
