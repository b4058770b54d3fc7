"""SPRT alarm flags (north_star "SPRT alarm flags must be bit-exact").

The reference has no SPRT: parity against the reference
is unpinned.  The definition (csrc/sprt.cuh, include/cstress_b200.h) is
pinned here in two steps: the C oracle against an independent pure-Python
loop (CPU), then the GPU's chunked speculate/fix-up scheme against the
oracle, bit for bit, including stream continuation and chunk-boundary cases.
"""
import math

import numpy as np
import pytest


def _resid(N, n, seed, shifts=()):
    rng = np.random.default_rng(seed)
    r = rng.standard_normal((N, n)) * np.linspace(0.5, 2.0, n)
    for (t0, t1, s, mu) in shifts:
        r[t0:t1, s] += mu
    return np.asfortranarray(r)


def _py_sprt(r, c, h, A, B, state):
    N, n = r.shape
    flags = np.zeros((N, n), dtype=np.uint8)
    st = state.copy()
    for s in range(n):
        lp, ln = st[s]
        for t in range(N):
            f = 0
            lp = lp + c[s] * (r[t, s] - h[s])
            if lp >= B:
                f |= 1
                lp = 0.0
            elif lp <= A:
                lp = 0.0
            ln = ln + c[s] * ((-r[t, s]) - h[s])
            if ln >= B:
                f |= 2
                ln = 0.0
            elif ln <= A:
                ln = 0.0
            flags[t, s] = f
        st[s] = (lp, ln)
    return flags, st


def test_oracle_sprt_matches_python_loop(oracle):
    sig = np.linspace(0.5, 2.0, 3)
    r = _resid(3000, 3, 1, [(1000, 1400, 1, 2.0), (2000, 2300, 2, -3.0)])
    c, h, A, B = oracle.sprt_params(sig, 3.0, 1e-3, 1e-3)
    flags, st, counts = oracle.sprt(r, c, h, A, B)
    want, wst = _py_sprt(r, c, h, A, B, np.zeros((3, 2)))
    assert np.array_equal(flags, want) and np.array_equal(st, wst)
    assert counts[1, 0] > 0 and counts[2, 1] > 0          # the injected shifts alarm
    assert np.array_equal(counts, np.stack([(flags & 1).sum(0), (flags >> 1 & 1).sum(0)], 1))
    assert math.isclose(A, math.log(1e-3 / (1 - 1e-3))) and math.isclose(B, -A)


def test_sprt_params_match_oracle(oracle):
    from paper_2003_08011_b200.sprt import sprt_params
    sig = np.array([0.3, 1.0, 7.5])
    for a, b in zip(sprt_params(sig, 2.5, 1e-2, 1e-4), oracle.sprt_params(sig, 2.5, 1e-2, 1e-4)):
        assert np.array_equal(np.asarray(a), np.asarray(b))


@pytest.fixture(scope="module")
def p():
    import torch  # noqa: F401
    import paper_2003_08011_b200 as p
    p.context(0)
    return p


@pytest.mark.gpu
@pytest.mark.parametrize("N,n,k,alpha", [
    (100_000, 7, 3.0, 1e-3), (257, 3, 3.0, 1e-3), (255, 1, 2.0, 1e-2), (1, 4, 3.0, 1e-3),
    (20_000, 5, 0.1, 1e-12),     # tiny drift, rare decisions: long fix-up re-runs
    (50_000, 3, 8.0, 1e-1)])     # frequent decisions
def test_gpu_sprt_bitwise(p, oracle, N, n, k, alpha):
    sig = np.linspace(0.5, 2.0, n)
    r = _resid(N, n, N + n, [(N // 3, N // 3 + 500, 0, 2.5), (N // 2, N // 2 + 300, n - 1, -2.0)])
    det = p.SprtDetector(sig, k, alpha, alpha)
    flags, counts = det.update(r)
    c, h, A, B = oracle.sprt_params(sig, k, alpha, alpha)
    want, st, wc = oracle.sprt(r, c, h, A, B)
    assert np.array_equal(flags, want)
    assert np.array_equal(det.state, st)
    assert np.array_equal(counts, wc)


@pytest.mark.gpu
def test_gpu_sprt_stream_continuation_and_device(p, oracle):
    import torch
    N, n = 60_000, 4
    sig = np.array([1.0, 0.5, 2.0, 1.5])
    r = _resid(N, n, 9, [(30_000, 31_000, 2, 5.0)])
    c, h, A, B = oracle.sprt_params(sig, 3.0, 1e-3, 1e-3)
    want, st, wc = oracle.sprt(r, c, h, A, B)
    det = p.SprtDetector(sig)
    parts = [det.update(r[a:b])[0] for a, b in [(0, 1000), (1000, 1001), (1001, 33_333), (33_333, N)]]
    assert np.array_equal(np.concatenate(parts), want)
    assert np.array_equal(det.state, st)
    # device residuals, FP32: the oracle sees the same (widened) values
    r32 = r.astype(np.float32)
    want32, st32, wc32 = oracle.sprt(r32.astype(np.float64), c, h, A, B)
    d = torch.tensor(r32.T.copy(), device="cuda").T
    det2 = p.SprtDetector(sig)
    flags, counts = det2.update_device(d)
    torch.cuda.synchronize()
    assert np.array_equal(flags.cpu().numpy(), want32)
    assert np.array_equal(counts, wc32) and np.array_equal(det2.state, st32)


@pytest.mark.gpu
def test_gpu_sprt_on_mset_residuals(p, oracle):
    """End to end: FP32 tensor-core surveillance residuals -> SPRT flags; a
    drift injected into one signal raises alarms there."""
    X = oracle.synthesize_uniform(10, 400, 0.5, 0.3, 1.0, 0.5, 4.0, 3)
    obs = oracle.synthesize_uniform(10, 5000, 0.5, 0.3, 1.0, 0.5, 4.0, 4)
    g = p.train(X, 100, p.KernelConfig(), p.BackendId("b200", 0, "fp32"))
    sigma = p.residual_sigma(p.estimate(g, X).residuals) + 1e-3
    drift = obs.copy()
    drift[2500:, 4] += 4.0 * obs[:, 4].std()
    r = p.estimate(g, drift).residuals
    flags, counts = p.SprtDetector(sigma, 3.0, 1e-3, 1e-3).update(r)
    c, h, A, B = oracle.sprt_params(sigma, 3.0, 1e-3, 1e-3)
    assert np.array_equal(flags, oracle.sprt(r, c, h, A, B)[0])
    assert counts[4].sum() == counts.sum(1).max() and counts[4].sum() > 10
