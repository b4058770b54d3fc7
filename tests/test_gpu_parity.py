"""GPU parity tests: the B200 path through the C-ABI against the CPU oracle.

Ports of test_mset.cpp / test_backends.cpp / acceptance.cpp criteria 1-2 with
the B200 backend in place of the reference's `optimized` backend, plus the
bit-exactness claims of this build:
  * sim_matrix (inverse distance) and matmul/batched_solve: bitwise equal to
    the reference loop nests;
  * select_memory_vectors: bitwise equal indices;
  * FP64 estimate given the same model: bitwise equal to the reference
    association and order;
  * FP32 (tcgen05 3xFP16) estimate: max|est - est_ref| <= 1e-3 max|est_ref|
    (north_star tolerance; typical 1e-6..1e-5).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-3   # north_star: "1e-3 FP32", relative to max |estimate|
FP64_TOL = 1e-10  # test_mset.cpp:264-278 cross-backend estimate tolerance


@pytest.fixture(scope="module")
def p():
    import torch  # noqa: F401  maps the CUDA math libraries cuSOLVER shares
    import paper_2003_08011_b200 as p
    p.context(0)  # fails loudly if the library or the device is missing
    # one-time cold start: the first eigendecomposition binds cuSOLVER
    p.symmetric_eig(np.eye(2), p.BackendId())
    return p


def B(p, precision="fp64"):
    return p.BackendId("b200", 0, precision)


def rel(got, want):
    return float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-300))


def max_rel_dev(got, want):
    return float((np.abs(got - want) / np.maximum(np.abs(want), 1e-300)).max()) if want.size else 0.0


# ----------------------------------------------------------------- per-op
def test_sim_matrix_bitwise_inverse_distance(p, oracle):
    rng = oracle.TestRng(0xC1)
    for i in range(40):
        n, pp, q = rng.uniform_int(1, 256), rng.uniform_int(1, 256), rng.uniform_int(1, 256)
        A = rng.matrix(n, pp, -1.0, 1.0)
        Bm = rng.matrix(n, q, -1.0, 1.0)
        got = p.sim_matrix(A, Bm, p.KernelConfig(), B(p))
        want = oracle.sim_matrix_reference(A, Bm)
        assert np.array_equal(got, want), (n, pp, q)


def test_sim_matrix_gaussian_and_edges(p, oracle):
    rng = oracle.TestRng(11)
    A = rng.matrix(16, 96, -1.0, 1.0)
    cfg = p.KernelConfig(p.KernelKind.gaussian)
    assert max_rel_dev(p.sim_matrix(A, A, cfg, B(p)),
                       oracle.sim_matrix_reference(A, A, oracle.GAUSSIAN)) <= 1e-14
    col = np.array([[1.0], [2.0], [3.0]])
    assert p.sim_matrix(col, col, p.KernelConfig(p.KernelKind.inverse_distance, 1.0), B(p))[0, 0] == 1.0
    assert p.sim_matrix(col, np.zeros((3, 0)), p.KernelConfig(), B(p)).shape == (1, 0)
    with pytest.raises(p.ShapeError):
        p.sim_matrix(A, np.zeros((2, 4)), p.KernelConfig(), B(p))
    # kernel symmetry sim(A,B) == sim(B,A)^T exactly (test_mset.cpp:158-160)
    X, Y = rng.matrix(3, 7, -1, 1), rng.matrix(3, 5, -1, 1)
    assert np.array_equal(p.sim_matrix(X, Y, p.KernelConfig(), B(p)),
                          p.sim_matrix(Y, X, p.KernelConfig(), B(p)).T)


def test_matmul_bitwise(p, oracle):
    A = np.array([[1.0, 2.0], [3.0, 4.0]])
    Bm = np.array([[5.0, 6.0], [7.0, 8.0]])
    assert np.array_equal(p.matmul(A, Bm, B(p)), [[19.0, 22.0], [43.0, 50.0]])
    rng = oracle.TestRng(17)
    M = rng.matrix(64, 64, -1.0, 1.0)
    assert np.array_equal(p.matmul(M, np.eye(64), B(p)), M)
    for _ in range(30):
        pp, m, q = rng.uniform_int(1, 256), rng.uniform_int(1, 256), rng.uniform_int(1, 256)
        X, Y = rng.matrix(pp, m, -1, 1), rng.matrix(m, q, -1, 1)
        assert np.array_equal(p.matmul(X, Y, B(p)), oracle.matmul_reference(X, Y))
    with pytest.raises(p.ShapeError):
        p.matmul(X, np.zeros((3, 4)), B(p))


def test_batched_solve_transparency(p, oracle):
    rng = oracle.TestRng(23)
    G = rng.matrix(20, 20, -1.0, 1.0)
    assert not p.batched_solve(G, np.zeros((20, 7)), B(p)).any()
    S = rng.matrix(20, 5, -1.0, 1.0)
    batch = p.batched_solve(G, S, B(p))
    for j in range(5):
        assert np.array_equal(batch[:, j:j + 1], p.batched_solve(G, S[:, j:j + 1], B(p)))
    assert np.array_equal(batch, oracle.matmul_reference(G, S))


def test_symmetric_eig_contract(p, oracle):
    e = p.symmetric_eig(np.eye(4), B(p))
    assert np.abs(e.eigenvalues - 1.0).max() < 1e-14
    assert np.linalg.norm(e.eigenvectors.T @ e.eigenvectors - np.eye(4)) <= 1e-9
    assert np.allclose(p.symmetric_eig(np.diag([3.0, 1.0, 2.0]), B(p)).eigenvalues, [1, 2, 3])
    g = oracle.TestRng(21).matrix(8, 8, -1.0, 1.0)
    g = 0.5 * (g + g.T)
    e = p.symmetric_eig(g, B(p))
    V, w = e.eigenvectors, e.eigenvalues
    gn = np.linalg.norm(g)
    assert np.linalg.norm(V @ np.diag(w) @ V.T - g) <= 1e-8 * gn
    assert np.linalg.norm(V.T @ V - np.eye(8)) <= 1e-9
    assert np.abs(oracle.jacobi_eig(g)[0] - w).max() < 1e-10
    with pytest.raises(p.ShapeError):
        p.symmetric_eig(np.array([[1.0, 0.5], [0.0, 1.0]]), B(p))


# -------------------------------------------------------------- selection
def test_selection_known_answers(p):
    mem = p.select_memory_vectors(np.array([[5.0], [-3.0], [9.0], [0.0]]), 2, B(p))
    assert sorted(mem.source_indices) == [1, 2]
    X = np.array([[-10.0, 1.0], [10.0, 2.0], [0.0, -5.0], [1.0, 5.0], [0.5, 0.5], [0.2, 0.1]])
    assert sorted(p.select_memory_vectors(X, 4, B(p)).source_indices) == [0, 1, 2, 3]
    X = np.array([[1.0, 0.0], [2.0, 1.0], [3.0, 2.0], [4.0, 3.0], [5.0, 4.0]])
    with pytest.raises(p.ConstraintViolated, match="m=3 violates m >= 2n with n=2"):
        p.select_memory_vectors(X, 3, B(p))
    with pytest.raises(p.InsufficientTraining):
        p.select_memory_vectors(X, 6, B(p))
    with pytest.raises(p.InsufficientTraining, match="distinct"):
        p.select_memory_vectors(np.array([[1.0], [1.0], [1.0], [1.0], [2.0], [3.0]]), 4, B(p))


@pytest.mark.parametrize("n,m", [(2, 6), (2, 25), (20, 100), (100, 1000), (1000, 4000)])
def test_selection_bitwise(p, oracle, n, m):
    if n == 2:
        X = oracle.TestRng(99).matrix(100, 2, -3.0, 3.0)
    else:
        X = oracle.synthesize_uniform(n, 4 * m, 0.5, 0.3, 1.0, 0.5, 4.0, 20260810)
    want_idx, want_D = oracle.select_memory_vectors(X, m)
    got = p.select_memory_vectors(X, m, B(p))
    assert got.source_indices == want_idx.tolist()
    assert np.array_equal(got.D, want_D)


def test_selection_ties_and_duplicates(p, oracle):
    X = np.round(oracle.TestRng(5).matrix(300, 3, -2.0, 2.0), 1)  # many ties / dupes
    for m in (6, 20, 40):
        want, _ = oracle.select_memory_vectors(X, m)
        assert p.select_memory_vectors(X, m, B(p)).source_indices == want.tolist()


# ------------------------------------------------------------------ train
def _sig(oracle, n, N, seed):
    return oracle.synthesize_uniform(n, N, 0.3, 0.2, 1.0, 0.2, 3.5, seed)


@pytest.mark.parametrize("kind", [0, 1])
def test_train_matches_oracle(p, oracle, kind):
    X = _sig(oracle, 8, 256, 37)
    cfg = p.KernelConfig(p.KernelKind(kind))
    g = p.train(X, 32, cfg, B(p))
    o = oracle.train(X, 32, kind)
    e = g.export()
    assert e["source_indices"].tolist() == o.source_indices.tolist()
    assert np.array_equal(e["D"], o.D)
    assert np.array_equal(e["signal_scale"], o.scale)  # sequential sums, bitwise
    assert g.rank == o.rank == 32
    assert np.abs(e["eigen_spectrum"] - o.eigen_spectrum).max() <= 1e-12 * o.eigen_spectrum.max()
    assert rel(e["gram_pinv"], o.gram_pinv) <= 1e-9
    gram = oracle.sim_matrix_reference(o.memory_normalized, o.memory_normalized, kind, o.h)
    assert np.abs(e["gram_pinv"] @ gram - np.eye(32)).max() < 1e-8


def test_training_unit_diagonal_full_rank_gaussian(p, oracle):
    # test_mset.cpp:201-226 against the B200 backend
    X = _sig(oracle, 2, 64, 31)
    model = p.train(X, 4, p.KernelConfig(p.KernelKind.gaussian), B(p))
    Dn = model.memory_normalized
    gram = p.sim_matrix(Dn, Dn, model.kernel, B(p))
    assert (np.diag(gram) == 1.0).all() and np.array_equal(gram, gram.T)
    assert model.rank == 4
    jw, _ = oracle.jacobi_eig(gram)
    assert np.abs(jw - model.eigen_spectrum).max() < 1e-10
    P = model.gram_pinv
    assert np.abs(P - P.T).max() <= 1e-12 * np.abs(P).max()
    assert np.abs(P @ gram - np.eye(4)).max() < 1e-8


def test_duplicate_rows_degrade_rank(p):
    model = p.train(np.array([[0.0], [1.0], [2.0], [3.0], [3.0]]), 4,
                    p.KernelConfig(p.KernelKind.gaussian, 1.0), B(p))
    assert model.rank < 4


def test_train_validates_inputs(p, oracle):
    X = _sig(oracle, 2, 32, 5)
    with pytest.raises(p.ConstraintViolated):
        p.train(X, 3, p.KernelConfig(), B(p))
    model = p.train(X, 4, p.KernelConfig(), B(p))
    with pytest.raises(p.ShapeError, match="observation signal count 3 does not match"):
        p.estimate(model, np.zeros((4, 3)))


# --------------------------------------------------------------- estimate
def test_fp64_estimate_bitwise_given_same_model(p, oracle):
    X = _sig(oracle, 8, 256, 37)
    obs = _sig(oracle, 8, 100, 41)
    for kind in (0, 1):
        o = oracle.train(X, 32, kind)
        gm = p.import_model(o.D, o.scale, o.gram_pinv, o.rank, p.KernelConfig(p.KernelKind(kind), o.h),
                            B(p))
        r = p.estimate(gm, obs)
        we, wr = oracle.estimate(o, obs)
        if kind == 0:
            assert np.array_equal(r.estimates, we) and np.array_equal(r.residuals, wr)
        else:  # CUDA exp vs glibc exp: last-ulp differences only
            assert rel(r.estimates, we) <= 1e-14


@pytest.mark.parametrize("kind", [0, 1])
def test_fp64_end_to_end_matches_oracle(p, oracle, kind):
    # acceptance criterion 1, end-to-end part (<= 1e-10)
    rng = oracle.TestRng(0xC1)
    for i in range(5):
        n = 8 if i == 0 else rng.uniform_int(2, 16)
        m = 32 if i == 0 else 2 * n + rng.uniform_int(0, 16)
        X = oracle.synthesize_uniform(n, 4 * m, 0.3, 0.2, 1.0, 0.2, 3.5, 1000 + i)
        obs = oracle.synthesize_uniform(n, 100, 0.3, 0.2, 1.0, 0.2, 3.5, 2000 + i)
        ref = oracle.estimate(oracle.train(X, m, kind), obs)[0]
        got = p.estimate(p.train(X, m, p.KernelConfig(p.KernelKind(kind)), B(p)), obs).estimates
        assert rel(got, ref) <= FP64_TOL


def test_memory_reproduction_fp64(p, oracle):
    # acceptance criterion 2 with the B200 backend
    rng = oracle.TestRng(0xC2)
    accepted = attempts = 0
    worst = 0.0
    while accepted < 20 and attempts < 200:
        attempts += 1
        n = rng.uniform_int(1, 16)
        m = rng.uniform_int(2 * n, 64)
        kind = p.KernelKind.inverse_distance if attempts % 2 == 0 else p.KernelKind.gaussian
        X = oracle.synthesize_uniform(n, 4 * m, 0.3, 0.2, 1.0, 0.2, 3.5, 3000 + attempts)
        model = p.train(X, m, p.KernelConfig(kind), B(p))
        if model.rank != m:
            continue
        accepted += 1
        res = p.estimate(model, model.memory.D.T.copy()).residuals
        worst = max(worst, float((np.abs(res).max(0) / model.signal_scale).max()))
    assert accepted == 20 and worst <= 1e-8


@pytest.mark.parametrize("n,m,N,kind", [
    (8, 32, 100, 0), (8, 32, 1000, 1), (20, 100, 1000, 0), (2, 4, 50, 0), (1, 2, 7, 1),
    (64, 512, 3000, 0), (100, 1000, 2000, 0), (100, 1000, 2000, 1), (120, 400, 700, 0),
    (140, 300, 300, 1), (33, 70, 129, 0),
    # large n: two-GEMM path (gemm_tc.cuh)
    (200, 500, 1000, 0), (257, 600, 700, 1), (131, 262, 129, 0), (512, 1024, 500, 0)])
def test_fp32_tensor_estimate_within_tolerance(p, oracle, n, m, N, kind):
    X = oracle.synthesize_uniform(n, 4 * m, 0.5, 0.3, 1.0, 0.5, 4.0, 77 + n)
    obs = oracle.synthesize_uniform(n, N, 0.5, 0.3, 1.0, 0.5, 4.0, 91 + n)
    o = oracle.train(X, m, kind)
    want_e, want_r = oracle.estimate(o, obs, oracle.OPTIMIZED, 64, 8)
    g = p.train(X, m, p.KernelConfig(p.KernelKind(kind)), B(p, "fp32"))
    r = p.estimate(g, obs)
    err = rel(r.estimates, want_e)
    print(f"n={n} m={m} N={N} kind={kind}: fp32 tensor rel err {err:.3e}")
    assert err <= FP32_TOL
    assert np.abs(r.residuals - (obs - r.estimates)).max() <= 1e-12 * np.abs(obs).max()


def test_fp32_memory_vectors_reproduce_themselves(p, oracle):
    X = _sig(oracle, 20, 400, 17)
    g = p.train(X, 100, p.KernelConfig(), B(p, "fp32"))
    res = p.estimate(g, g.memory.D.T.copy()).residuals
    assert (np.abs(res).max(0) / g.signal_scale).max() <= FP32_TOL


def test_constant_stream_finite(p, oracle):
    for prec in ("fp64", "fp32"):
        g = p.train(_sig(oracle, 3, 64, 13), 8, p.KernelConfig(), B(p, prec))
        r = p.estimate(g, np.full((10, 3), 4.2))
        assert np.isfinite(r.estimates).all() and np.isfinite(r.residuals).all()


def test_empty_observation_batch(p, oracle):
    g = p.train(_sig(oracle, 3, 64, 13), 8, p.KernelConfig(), B(p, "fp32"))
    r = p.estimate(g, np.zeros((0, 3)))
    assert r.estimates.shape == (0, 3)


def test_device_resident_estimate(p, oracle):
    import torch
    n, m, N = 20, 100, 5000
    X = oracle.synthesize_uniform(n, 4 * m, 0.5, 0.3, 1.0, 0.5, 4.0, 3)
    obs = oracle.synthesize_uniform(n, N, 0.5, 0.3, 1.0, 0.5, 4.0, 4)
    g = p.train(X, m, p.KernelConfig(), B(p, "fp32"))
    want = p.estimate(g, obs).estimates
    for dt in (torch.float32, torch.float64):
        d_obs = torch.tensor(obs.T.copy(), dtype=dt, device="cuda").T  # column-major
        d_est = torch.empty_like(d_obs.T).T
        d_res = torch.empty_like(d_obs.T).T
        p.estimate_device(g, d_obs, d_est, d_res)
        torch.cuda.synchronize()
        got = d_est.double().cpu().numpy()
        assert rel(got, want) <= (1e-6 if dt == torch.float32 else 1e-12)
        assert torch.allclose(d_res, d_obs - d_est)


def test_plugin_contract(p, oracle):
    X = _sig(oracle, 2, 64, 61)
    obs = _sig(oracle, 2, 16, 67)
    for name in ("mset2", "mean"):
        algo = p.algorithm_by_name(name)
        model = algo.train(X, 4, p.KernelConfig(), B(p))
        r = algo.estimate(model, obs, B(p))
        assert r.estimates.shape == obs.shape and np.isfinite(r.residuals).all()
    mean_model = p.algorithm_by_name("mean").train(X, 4, p.KernelConfig(), B(p))
    with pytest.raises(p.ConfigError, match="not trained by algorithm mset2"):
        p.algorithm_by_name("mset2").estimate(mean_model, obs, B(p))


def test_c2_full_size_fp32_properties(p, oracle):
    """BASELINE config 2 at full size (n=100, N=100k, m=1000): finite outputs,
    residual identity, and a 400-observation sample against the oracle."""
    import paper_2003_08011_b200 as pk
    X = pk.synthesize(pk.SignalSpec.uniform(100, 4000, 0.5, 0.3, 1.0, 0.5, 4.0, 11)).data
    obs = pk.synthesize(pk.SignalSpec.uniform(100, 100000, 0.5, 0.3, 1.0, 0.5, 4.0, 12)).data
    g = p.train(X, 1000, p.KernelConfig(), B(p, "fp32"))
    r = p.estimate(g, obs)
    assert np.isfinite(r.estimates).all()
    assert np.array_equal(r.residuals, obs - r.estimates)
    sel = np.random.default_rng(0).choice(100000, 400, replace=False)
    o = oracle.train(X, 1000, 0, backend=oracle.OPTIMIZED, tile=64, workers=8)
    want = oracle.estimate(o, obs[sel], oracle.OPTIMIZED, 64, 8)[0]
    assert rel(r.estimates[sel], want) <= FP32_TOL


def test_large_n_device_resident_and_c3_shape(p, oracle):
    """Two-GEMM path at BASELINE config 3's model shape (n=1000, m=4000):
    FP32 device-resident I/O and FP64 host I/O against the FP64 GPU estimate
    of the same model (bit-exact to the reference order, see
    test_fp64_estimate_bitwise_given_same_model) on a sample."""
    import torch
    import paper_2003_08011_b200 as pk
    n, m, N = 1000, 4000, 20000
    X = pk.synthesize(pk.SignalSpec.uniform(n, 4 * m, 0.5, 0.3, 1.0, 0.5, 4.0, 5)).data
    obs = pk.synthesize(pk.SignalSpec.uniform(n, N, 0.5, 0.3, 1.0, 0.5, 4.0, 6)).data
    g32 = p.train(X, m, p.KernelConfig(), B(p, "fp32"))
    g64 = p.train(X, m, p.KernelConfig(), B(p, "fp64"))
    sel = np.random.default_rng(1).choice(N, 512, replace=False)
    want = p.estimate(g64, obs[sel]).estimates
    r = p.estimate(g32, obs)
    assert np.isfinite(r.estimates).all()
    assert rel(r.estimates[sel], want) <= FP32_TOL
    d_obs = torch.tensor(obs.T.copy(), dtype=torch.float32, device="cuda").T
    d_est = torch.empty_like(d_obs.T).T
    d_res = torch.empty_like(d_obs.T).T
    p.estimate_device(g32, d_obs, d_est, d_res)
    torch.cuda.synchronize()
    got = d_est.double().cpu().numpy()
    assert rel(got[sel], want) <= FP32_TOL
    assert torch.allclose(d_res, d_obs - d_est)


def test_cpp_host_layer_on_gpu(p):
    """C++ ports of test_mset.cpp / test_backends.cpp through the C++ host layer."""
    import subprocess
    from paper_2003_08011_b200 import build as b
    r = subprocess.run([b.build_cpp_test()], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("split", ["0", "1"])
@pytest.mark.parametrize("n,m,N", [(100, 1000, 1000), (20, 100, 4000), (64, 512, 3000), (33, 70, 1024),
                                   (100, 1000, 148 * 128 * 2 + 5)])
def test_staged_readout_matches_direct_stores(p, oracle, n, m, N, split):
    """FP32 device I/O: the staged tile edge (x tiles arrive by TMA, estimates
    and residuals leave through shared memory and two tensor stores per tile,
    partial last tile included) against the plain path (global loads and
    stores).  The staged edge may sum ||x||^2 in a different order (split
    between the two epilogue sets), so the two agree to FP32 rounding, and
    each keeps residual = x - estimate exactly."""
    import os
    import torch
    X = oracle.synthesize_uniform(n, 4 * m, 0.5, 0.3, 1.0, 0.5, 4.0, 5 + n)
    obs = oracle.synthesize_uniform(n, N, 0.5, 0.3, 1.0, 0.5, 4.0, 6 + n)
    g = p.train(X, m, p.KernelConfig(), B(p, "fp32"))
    d_obs = torch.tensor(obs.T.copy(), dtype=torch.float32, device="cuda").T
    out = {}
    for staged in ("1", "0"):
        os.environ["CSB_STAGED_READOUT"] = staged
        os.environ["CSB_SPLIT_EDGE"] = split
        try:
            e = torch.full_like(d_obs.T, float("nan")).T
            r = torch.full_like(d_obs.T, float("nan")).T
            p.estimate_device(g, d_obs, e, r)
            torch.cuda.synchronize()
            out[staged] = (e.cpu().numpy(), r.cpu().numpy())
        finally:
            del os.environ["CSB_STAGED_READOUT"]
            del os.environ["CSB_SPLIT_EDGE"]
    assert np.isfinite(out["1"][0]).all() and np.isfinite(out["1"][1]).all()
    assert rel(out["1"][0], out["0"][0]) <= 1e-5
    x = obs.astype(np.float32)
    for k in ("1", "0"):
        assert np.array_equal(out[k][1], x - out[k][0])
    want = p.estimate(g, obs).estimates
    assert rel(out["1"][0].astype(np.float64), want) <= 1e-5


@pytest.mark.timeout(300)
@pytest.mark.parametrize("shape", ["64,2,2", "64,2,1", "64,1,1", "32,2,2", "128,1,1"])
@pytest.mark.parametrize("n,m", [(20, 64), (20, 100), (24, 150), (100, 1000)])
def test_fused_many_tiles_per_cta(p, oracle, shape, n, m):
    """Fused kernel with several observation tiles per CTA (148 persistent
    CTAs, >= 3 tiles each) for every (MT, NB, SB) TMEM plan and 1..16 memory
    tiles per observation tile: the tile-boundary hand-offs (x prologue,
    ||x||^2 hand-over, O readout) must neither deadlock nor mix tiles.
    Checked against the GPU FP64 estimate (bitwise the reference order) of
    the same training data, and a sample against the oracle."""
    import os
    N = 148 * 128 * 3 + 77
    X = oracle.synthesize_uniform(n, 4 * m, 0.5, 0.3, 1.0, 0.5, 4.0, 31 + n)
    obs = oracle.synthesize_uniform(n, N, 0.5, 0.3, 1.0, 0.5, 4.0, 37 + n)
    os.environ["CSB_TC_SHAPE"] = shape
    try:
        g = p.train(X, m, p.KernelConfig(), B(p, "fp32"))
    finally:
        del os.environ["CSB_TC_SHAPE"]
    g64 = p.train(X, m, p.KernelConfig(), B(p, "fp64"))
    want = p.estimate(g64, obs).estimates
    r = p.estimate(g, obs)
    assert rel(r.estimates, want) <= FP32_TOL
    assert np.array_equal(r.residuals, obs - r.estimates)
    sel = np.arange(0, N, 997)
    o = oracle.train(X, m, 0)
    assert rel(r.estimates[sel], oracle.estimate(o, obs[sel])[0]) <= FP32_TOL


@pytest.mark.timeout(300)
@pytest.mark.parametrize("cluster", ["2", "4"])
def test_fused_cluster_multicast(p, oracle, cluster):
    """CSB_CLUSTER=2|4: CTA clusters share the D_norm / P operand stream by
    multicast bulk copies (each CTA loads a 1/CL slice into every CTA of the
    cluster; slots freed by multicast MMA commits).  Same results as the
    plain launch, including dummy tile slots when the tile count is not a
    multiple of the cluster size."""
    import os
    import torch
    n, m, N = 100, 1000, 128 * (148 * 2 + 3) + 11
    X = oracle.synthesize_uniform(n, 4 * m, 0.5, 0.3, 1.0, 0.5, 4.0, 51)
    obs = oracle.synthesize_uniform(n, N, 0.5, 0.3, 1.0, 0.5, 4.0, 53)
    g = p.train(X, m, p.KernelConfig(), B(p, "fp32"))
    d_obs = torch.tensor(obs.T.astype(np.float32), device="cuda").T
    out = {}
    for cl in ("1", cluster):
        os.environ["CSB_CLUSTER"] = cl
        try:
            e = torch.full_like(d_obs.T, float("nan")).T
            r = torch.full_like(d_obs.T, float("nan")).T
            p.estimate_device(g, d_obs, e, r)
            torch.cuda.synchronize()
            out[cl] = (e.cpu().numpy(), r.cpu().numpy())
        finally:
            del os.environ["CSB_CLUSTER"]
    assert np.array_equal(out["1"][0], out[cluster][0]) and np.array_equal(out["1"][1], out[cluster][1])
