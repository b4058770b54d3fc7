"""Pins the CPU oracle to the reference's own tests (CPU only, no GPU).

Ports of /root/reference/proj/tests/test_mset.cpp and test_backends.cpp:
the known-answer tests verbatim and the relational pins with the reference's
tolerances.  The oracle is the checker for every GPU parity test, so it must
pass the reference's suite first.
"""
import math

import numpy as np
import pytest


def random_signals(o, n, N, seed):
    # test_mset.cpp:70-72
    return o.synthesize_uniform(n, N, 0.3, 0.2, 1.0, 0.2, 3.5, seed)


def selection_oracle(data, m):
    """Independent pure-Python restatement of test_mset.cpp:33-68."""
    N, n = data.shape
    chosen = [False] * N
    picked = []
    for s in range(n):
        imin = imax = 0
        for r in range(1, N):
            if data[r, s] < data[imin, s]:
                imin = r
            if data[r, s] > data[imax, s]:
                imax = r
        for idx in (imin, imax):
            if not chosen[idx]:
                chosen[idx] = True
                picked.append(idx)
    k = m - len(picked)
    pool = []
    for r in range(N):
        if chosen[r]:
            continue
        norm2 = 0.0
        for s in range(n):
            norm2 += float(data[r, s]) * float(data[r, s])
        pool.append((math.sqrt(norm2), r))
    pool.sort()
    u = len(pool)
    for i in range(k):
        pos = (u - 1) // 2 if k == 1 else i * (u - 1) // (k - 1)
        picked.append(pool[pos][1])
    return picked


def test_splitmix64_known_answer(oracle):
    # SplitMix64 (Steele, Lea & Flood 2014) published first output for seed 0
    assert oracle.splitmix64_mix(0) == 0xE220A8397B1DCDAF


def test_kernel_eval_closed_forms(oracle):
    # test_mset.cpp:76-94
    assert oracle.kernel_from_d2(0.0, oracle.GAUSSIAN, 1.0) == 1.0
    assert oracle.kernel_from_d2(0.0, oracle.INVERSE_DISTANCE, 2.0) == 1.0
    g = oracle.kernel_from_d2(1.0, oracle.GAUSSIAN, 1.0)
    assert abs(g - math.exp(-0.5)) <= 1e-12 * math.exp(-0.5)
    assert abs(g - 0.606531) <= 1e-6
    assert abs(oracle.kernel_from_d2(4.0, oracle.INVERSE_DISTANCE, 2.0) - 0.5) <= 1e-12


def test_selection_single_signal_extrema(oracle):
    # test_mset.cpp:96-107
    idx, D = oracle.select_memory_vectors(np.array([[5.0], [-3.0], [9.0], [0.0]]), 2)
    assert sorted(D[0].tolist()) == [-3.0, 9.0]
    assert sorted(idx.tolist()) == [1, 2]


def test_selection_stage1_fills_exactly(oracle):
    # test_mset.cpp:109-123
    X = np.array([[-10.0, 1.0], [10.0, 2.0], [0.0, -5.0], [1.0, 5.0], [0.5, 0.5], [0.2, 0.1]])
    idx, _ = oracle.select_memory_vectors(X, 4)
    assert sorted(idx.tolist()) == [0, 1, 2, 3]


@pytest.mark.parametrize("m", [6, 25])
def test_selection_stage2_stride_oracle(oracle, m):
    # test_mset.cpp:125-135
    X = oracle.TestRng(99).matrix(100, 2, -3.0, 3.0)
    idx, _ = oracle.select_memory_vectors(X, m)
    assert idx.tolist() == selection_oracle(X, m)


def test_selection_preconditions(oracle):
    # test_mset.cpp:137-147
    X = np.array([[1.0, 0.0], [2.0, 1.0], [3.0, 2.0], [4.0, 3.0], [5.0, 4.0]])
    with pytest.raises(oracle.OracleError) as e:
        oracle.select_memory_vectors(X, 3)
    assert e.value.kind == "ConstraintViolated"
    assert str(e.value) == "select_memory_vectors: m=3 violates m >= 2n with n=2"
    with pytest.raises(oracle.OracleError) as e:
        oracle.select_memory_vectors(X, 6)
    assert e.value.kind == "InsufficientTraining"
    dupes = np.array([[1.0], [1.0], [1.0], [1.0], [2.0], [3.0]])
    with pytest.raises(oracle.OracleError) as e:
        oracle.select_memory_vectors(dupes, 4)
    assert e.value.kind == "InsufficientTraining"


def test_similarity_matches_naive_and_is_symmetric(oracle):
    # test_mset.cpp:149-161
    rng = oracle.TestRng(7)
    A = rng.matrix(3, 2, -1.0, 1.0)
    B = rng.matrix(3, 2, -1.0, 1.0)
    got = oracle.sim_matrix_reference(A, B, oracle.GAUSSIAN, 1.3)
    d2 = ((A[:, :, None] - B[:, None, :]) ** 2).sum(0)
    want = np.exp(-d2 / (2 * 1.3 * 1.3))
    assert np.abs(got - want).max() <= 1e-14
    ba = oracle.sim_matrix_reference(B, A, oracle.GAUSSIAN, 1.3)
    assert np.array_equal(got, ba.T)


def test_symmetric_eig_contract(oracle):
    # test_mset.cpp:163-199
    w, V = oracle.symmetric_eig(np.eye(4))
    assert np.abs(w - 1.0).max() < 1e-14
    assert np.linalg.norm(V.T @ V - np.eye(4)) <= 1e-9
    w, _ = oracle.symmetric_eig(np.diag([3.0, 1.0, 2.0]))
    assert np.allclose(w, [1.0, 2.0, 3.0])
    g = oracle.TestRng(21).matrix(8, 8, -1.0, 1.0)
    g = 0.5 * (g + g.T)
    w, V = oracle.symmetric_eig(g)
    gn = np.linalg.norm(g)
    assert np.linalg.norm(V @ np.diag(w) @ V.T - g) <= 1e-8 * gn
    assert np.linalg.norm(g @ V - V @ np.diag(w)) <= 1e-8 * gn
    assert np.linalg.norm(V.T @ V - np.eye(8)) <= 1e-9
    jw, _ = oracle.jacobi_eig(g)
    assert np.abs(jw - w).max() < 1e-10
    with pytest.raises(oracle.OracleError) as e:
        oracle.symmetric_eig(np.array([[1.0, 0.5], [0.0, 1.0]]))
    assert e.value.kind == "ShapeError"


def test_symmetric_eig_large_matches_numpy(oracle):
    g = oracle.TestRng(5).matrix(200, 200, -1.0, 1.0)
    g = 0.5 * (g + g.T)
    w, V = oracle.symmetric_eig(g)
    assert np.abs(w - np.linalg.eigvalsh(g)).max() < 1e-12
    assert np.linalg.norm(g @ V - V * w) <= 1e-8 * np.linalg.norm(g)


def test_training_unit_diagonal_full_rank_gaussian(oracle):
    # test_mset.cpp:201-226
    X = random_signals(oracle, 2, 64, 31)
    model = oracle.train(X, 4, oracle.GAUSSIAN)
    gram = oracle.sim_matrix_reference(model.memory_normalized, model.memory_normalized,
                                       oracle.GAUSSIAN, model.h)
    assert (np.diag(gram) == 1.0).all()
    assert np.array_equal(gram, gram.T)
    assert model.rank == 4
    jw, _ = oracle.jacobi_eig(gram)
    assert jw.min() > 0.0
    assert np.abs(jw - model.eigen_spectrum).max() < 1e-10
    P = model.gram_pinv
    assert np.abs(P - P.T).max() <= 1e-12 * np.abs(P).max()
    assert np.abs(P @ gram - np.eye(4)).max() < 1e-8


def test_duplicate_rows_degrade_rank(oracle):
    # test_mset.cpp:228-234
    model = oracle.train(np.array([[0.0], [1.0], [2.0], [3.0], [3.0]]), 4, oracle.GAUSSIAN, 1.0)
    assert model.rank < 4


def test_memory_vectors_reproduce_themselves(oracle):
    # test_mset.cpp:236-250
    X = random_signals(oracle, 2, 128, 17)
    model = oracle.train(X, 4, oracle.INVERSE_DISTANCE)
    assert model.rank == 4
    _, res = oracle.estimate(model, model.D.T.copy())
    for s in range(2):
        assert np.abs(res[:, s]).max() <= 1e-8 * model.scale[s]


def test_constant_stream_stays_finite(oracle):
    # test_mset.cpp:252-262
    model = oracle.train(random_signals(oracle, 3, 64, 13), 8)
    est, res = oracle.estimate(model, np.full((10, 3), 4.2))
    assert np.isfinite(est).all() and np.isfinite(res).all()


def test_estimate_agrees_across_backends(oracle):
    # test_mset.cpp:264-278
    X = random_signals(oracle, 8, 256, 37)
    obs = random_signals(oracle, 8, 100, 41)
    a = oracle.estimate(oracle.train(X, 32), obs)[0]
    mo = oracle.train(X, 32, backend=oracle.OPTIMIZED, tile=16, workers=2)
    b = oracle.estimate(mo, obs, oracle.OPTIMIZED, 16, 2)[0]
    assert np.abs(a - b).max() <= 1e-10 * np.abs(a).max()


def test_train_estimate_validate_inputs(oracle):
    # test_mset.cpp:280-290
    X = random_signals(oracle, 2, 32, 5)
    with pytest.raises(oracle.OracleError) as e:
        oracle.train(X, 3)
    assert e.value.kind == "ConstraintViolated"
    model = oracle.train(X, 4)
    with pytest.raises(oracle.OracleError) as e:
        oracle.estimate(model, np.zeros((4, 3)))
    assert e.value.kind == "ShapeError"


def max_rel_dev(got, want):
    # test_backends.cpp:13-22
    return float((np.abs(got - want) / np.maximum(np.abs(want), 1e-300)).max()) if want.size else 0.0


def test_reference_similarity_basics(oracle):
    # test_backends.cpp:32-58
    col = np.array([[1.0], [2.0], [3.0]])
    assert oracle.sim_matrix_reference(col, col, oracle.INVERSE_DISTANCE, 1.0)[0, 0] == 1.0
    assert oracle.sim_matrix_reference(col, np.zeros((3, 0))).shape == (1, 0)
    assert oracle.sim_matrix_reference(np.zeros((3, 0)), np.zeros((3, 0))).size == 0
    rng = oracle.TestRng(3)
    A = rng.matrix(3, 4, -2.0, 2.0)
    B = rng.matrix(3, 5, -2.0, 2.0)
    got = oracle.sim_matrix_reference(A, B, oracle.INVERSE_DISTANCE, 1.0)
    d = np.sqrt(((A[:, :, None] - B[:, None, :]) ** 2).sum(0))
    assert np.abs(got - 1.0 / (1.0 + d)).max() <= 1e-15
    with pytest.raises(oracle.OracleError):
        oracle.sim_matrix_reference(A, np.zeros((2, 4)))


def test_optimized_similarity_matches_reference(oracle):
    # test_backends.cpp:60-97
    rng = oracle.TestRng(11)
    A, B = rng.matrix(5, 17, -1.0, 1.0), rng.matrix(5, 13, -1.0, 1.0)
    assert max_rel_dev(oracle.sim_matrix_optimized(A, B, tile=32, workers=1),
                       oracle.sim_matrix_reference(A, B)) <= 1e-14
    A, B = rng.matrix(64, 512, -1.0, 1.0), rng.matrix(64, 512, -1.0, 1.0)
    assert max_rel_dev(oracle.sim_matrix_optimized(A, B, tile=64, workers=4),
                       oracle.sim_matrix_reference(A, B)) <= 1e-12
    A, B = rng.matrix(33, 130, -1.0, 1.0), rng.matrix(33, 70, -1.0, 1.0)
    w1 = oracle.sim_matrix_optimized(A, B, tile=16, workers=1)
    assert np.array_equal(w1, oracle.sim_matrix_optimized(A, B, tile=16, workers=2))
    assert np.array_equal(w1, oracle.sim_matrix_optimized(A, B, tile=16, workers=8))
    A = rng.matrix(16, 96, -1.0, 1.0)
    assert max_rel_dev(oracle.sim_matrix_optimized(A, A, oracle.GAUSSIAN, tile=24, workers=3),
                       oracle.sim_matrix_reference(A, A, oracle.GAUSSIAN)) <= 1e-12


def test_matmul_known_answer_and_oracle(oracle):
    # test_backends.cpp:99-121
    A = np.array([[1.0, 2.0], [3.0, 4.0]])
    B = np.array([[5.0, 6.0], [7.0, 8.0]])
    want = np.array([[19.0, 22.0], [43.0, 50.0]])
    assert np.array_equal(oracle.matmul_reference(A, B), want)
    assert np.array_equal(oracle.matmul_optimized(A, B, tile=8, workers=2), want)
    rng = oracle.TestRng(17)
    M = rng.matrix(64, 64, -1.0, 1.0)
    assert np.array_equal(oracle.matmul_reference(M, np.eye(64)), M)
    X, Y = rng.matrix(64, 48, -1.0, 1.0), rng.matrix(48, 56, -1.0, 1.0)
    ref = oracle.matmul_reference(X, Y)
    assert max_rel_dev(oracle.matmul_optimized(X, Y, tile=16, workers=3), ref) <= 1e-12
    assert np.abs(ref - X @ Y).max() <= 1e-12
    with pytest.raises(oracle.OracleError):
        oracle.matmul_reference(X, np.zeros((3, 4)))


def test_batched_solve_transparency(oracle):
    # test_backends.cpp:123-141 (batched_solve == matmul(G_pinv, S))
    rng = oracle.TestRng(23)
    G = rng.matrix(20, 20, -1.0, 1.0)
    assert not oracle.matmul_reference(G, np.zeros((20, 7))).any()
    S = rng.matrix(20, 5, -1.0, 1.0)
    batch = oracle.matmul_optimized(G, S, tile=8, workers=2)
    for j in range(5):
        single = oracle.matmul_optimized(G, S[:, j:j + 1], tile=8, workers=2)
        assert np.array_equal(batch[:, j:j + 1], single)
    assert max_rel_dev(batch, oracle.matmul_reference(G, S)) <= 1e-12


def test_randomized_oracle_equivalence(oracle):
    # test_backends.cpp:143-157
    rng = oracle.TestRng(31)
    for _ in range(10):
        n, p, q = rng.uniform_int(1, 96), rng.uniform_int(1, 96), rng.uniform_int(1, 96)
        A = rng.matrix(n, p, -1.0, 1.0)
        B = rng.matrix(n, q, -1.0, 1.0)
        tile, workers = rng.uniform_int(8, 64), rng.uniform_int(1, 4)
        assert max_rel_dev(oracle.sim_matrix_optimized(A, B, tile=tile, workers=workers),
                           oracle.sim_matrix_reference(A, B)) <= 1e-12


def test_backend_validation(oracle):
    # test_backends.cpp:159-171 (tile / worker bounds)
    A = np.ones((2, 2))
    for tile, workers in [(4, 1), (2048, 1), (64, -1)]:
        with pytest.raises(oracle.OracleError) as e:
            oracle.sim_matrix_optimized(A, A, tile=tile, workers=workers)
        assert e.value.kind == "ConfigError"
