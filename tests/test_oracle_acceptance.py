"""Reference acceptance criteria 1, 2, 3 and the signal-synthesis pins,
run against the CPU oracle (acceptance.cpp:74-187, test_signals.cpp)."""
import numpy as np
import pytest


def max_rel_dev(got, want):
    if want.size == 0:
        return 0.0
    return float((np.abs(got - want) / np.maximum(np.abs(want), 1e-300)).max())


def test_criterion1_oracle_equivalence(oracle):
    # acceptance.cpp:74-131
    rng = oracle.TestRng(0xC1)
    worst_sim = worst_mm = worst_e2e = 0.0
    for i in range(100):
        n, p, q = rng.uniform_int(1, 256), rng.uniform_int(1, 256), rng.uniform_int(1, 256)
        A = rng.matrix(n, p, -1.0, 1.0)
        B = rng.matrix(n, q, -1.0, 1.0)
        kind = oracle.INVERSE_DISTANCE if i % 2 == 0 else oracle.GAUSSIAN
        tile, workers = rng.uniform_int(8, 256), rng.uniform_int(1, 8)
        worst_sim = max(worst_sim, max_rel_dev(
            oracle.sim_matrix_optimized(A, B, kind, 0.0, tile, workers),
            oracle.sim_matrix_reference(A, B, kind)))
    for _ in range(100):
        p, m, q = rng.uniform_int(1, 256), rng.uniform_int(1, 256), rng.uniform_int(1, 256)
        A = rng.matrix(p, m, -1.0, 1.0)
        B = rng.matrix(m, q, -1.0, 1.0)
        workers, tile = rng.uniform_int(1, 8), rng.uniform_int(8, 256)
        worst_mm = max(worst_mm, max_rel_dev(oracle.matmul_optimized(A, B, tile, workers),
                                             oracle.matmul_reference(A, B)))
    for i in range(5):
        n = 8 if i == 0 else rng.uniform_int(2, 16)
        m = 32 if i == 0 else 2 * n + rng.uniform_int(0, 16)
        X = oracle.synthesize_uniform(n, 4 * m, 0.3, 0.2, 1.0, 0.2, 3.5, 1000 + i)
        obs = oracle.synthesize_uniform(n, 100, 0.3, 0.2, 1.0, 0.2, 3.5, 2000 + i)
        kind = oracle.INVERSE_DISTANCE if i % 2 == 0 else oracle.GAUSSIAN
        ref = oracle.estimate(oracle.train(X, m, kind), obs)[0]
        mo = oracle.train(X, m, kind, backend=oracle.OPTIMIZED, tile=32, workers=2)
        fast = oracle.estimate(mo, obs, oracle.OPTIMIZED, 32, 2)[0]
        worst_e2e = max(worst_e2e, np.abs(ref - fast).max() / np.abs(ref).max())
    assert worst_sim <= 1e-12 and worst_mm <= 1e-12 and worst_e2e <= 1e-10


def test_criterion2_memory_reproduction(oracle):
    # acceptance.cpp:133-165
    rng = oracle.TestRng(0xC2)
    accepted = attempts = 0
    worst = 0.0
    while accepted < 50 and attempts < 500:
        attempts += 1
        n = rng.uniform_int(1, 16)
        m = rng.uniform_int(2 * n, 64)
        kind = oracle.INVERSE_DISTANCE if attempts % 2 == 0 else oracle.GAUSSIAN
        X = oracle.synthesize_uniform(n, 4 * m, 0.3, 0.2, 1.0, 0.2, 3.5, 3000 + attempts)
        model = oracle.train(X, m, kind)
        if model.rank != m:
            continue
        accepted += 1
        _, res = oracle.estimate(model, model.D.T.copy())
        worst = max(worst, float((np.abs(res).max(0) / model.scale).max()))
    assert accepted == 50 and worst <= 1e-8


def test_criterion3_constraint_holes(oracle):
    # acceptance.cpp:167-187
    cells = oracle.generate_cells([32 << k for k in range(6)], [1024],
                                  [128 << k for k in range(7)])
    assert len(cells) == 42
    excluded = 0
    for (n, _, m), ok in cells:
        assert ok == (m >= 2 * n)
        excluded += not ok
    assert excluded > 0


def test_cell_order_and_seeds(oracle):
    # test_sweep.cpp:48-59, :91-120
    cells = oracle.generate_cells([1, 2], [10, 20], [4, 8])
    assert [c[0] for c in cells][:5] == [(1, 10, 4), (1, 20, 4), (1, 10, 8), (1, 20, 8), (2, 10, 4)]
    a0 = oracle.cell_data_seed(9, 2, 32, 4, 0)
    assert a0 == oracle.cell_data_seed(9, 2, 32, 4, 0)
    assert a0 != oracle.cell_data_seed(9, 2, 32, 4, 1)
    assert a0 != oracle.cell_data_seed(10, 2, 32, 4, 0)
    assert a0 == oracle.derive_seed(9, [2, 32, 4, 0])


def _moments(x):
    x = x - x.mean()
    m2 = (x * x).mean()
    return m2, (x ** 3).mean() / m2 ** 1.5, (x ** 4).mean() / m2 ** 2


def test_fleishman_quadrature_and_infeasible(oracle):
    # test_signals.cpp:42-60
    z, w = np.polynomial.hermite_e.hermegauss(80)
    w = w / w.sum()
    for skew, kurt in [(0.5, 4.0), (1.0, 5.0), (-0.8, 4.5), (0.0, 3.0)]:
        a, b, c, d = oracle.solve_fleishman(skew, kurt)
        y = a + b * z + c * z * z + d * z ** 3
        m1 = (w * y).sum()
        yc = y - m1
        m2, m3, m4 = (w * yc ** 2).sum(), (w * yc ** 3).sum(), (w * yc ** 4).sum()
        assert abs(m1) < 1e-8 and abs(m2 - 1.0) < 1e-7
        assert abs(m3 / m2 ** 1.5 - skew) <= 5e-6 * max(abs(skew), 1e-300) + 1e-9
        assert abs(m4 / m2 ** 2 - kurt) <= 5e-6 * kurt
    with pytest.raises(oracle.OracleError) as e:
        oracle.solve_fleishman(2.0, 6.0)
    assert e.value.kind == "MomentInfeasible"


def test_synthesis_statistics(oracle):
    # test_signals.cpp:62-125 and acceptance criterion 7
    x = oracle.synthesize_uniform(1, 100000, 0.0, 0.0, 1.0, 0.0, 3.0, 7)[:, 0]
    m2, sk, ku = _moments(x)
    assert abs(sk) < 0.05 and 2.85 < ku < 3.15 and abs(m2 - 1.0) < 1e-9
    a = oracle.synthesize_uniform(3, 5000, 0.4, 0.2, 2.0, 0.5, 4.0, 42)
    b = oracle.synthesize_uniform(3, 5000, 0.4, 0.2, 2.0, 0.5, 4.0, 42)
    assert a.tobytes() == b.tobytes()
    m = oracle.synthesize_uniform(2, 200000, 0.8, 0.9, 1.0, 0.0, 3.0, 11)
    assert 0.85 < np.corrcoef(m[:, 0], m[:, 1])[0, 1] < 0.95
    for s in range(2):
        c = m[:, s] - m[:, s].mean()
        lag1 = (c[:-1] * c[1:]).sum() / (c * c).sum()
        assert 0.75 < lag1 < 0.85
    m = oracle.synthesize_uniform(2, 100000, 0.8, 0.9, 1.0, 1.0, 5.0, 20260810)
    for s in range(2):
        _, sk, ku = _moments(m[:, s])
        assert abs(sk - 1.0) <= 0.15 and abs(ku - 5.0) <= 0.6


def test_psd_repair_ladder(oracle):
    # test_signals.cpp:171-192
    r, jit = oracle.nearest_psd_repair(np.eye(3), 1e-6)
    assert jit == 0.0 and np.array_equal(r, np.eye(3))
    r, jit = oracle.nearest_psd_repair(np.array([[1.0, 1.0], [1.0, 1.0]]), 1e-6)
    assert jit <= 1e-8
    np.linalg.cholesky(r)
    with pytest.raises(oracle.OracleError) as e:
        oracle.nearest_psd_repair(np.array([[1.0, 1.5], [1.5, 1.0]]), 1e-6)
    assert e.value.kind == "BadCorrelation"
