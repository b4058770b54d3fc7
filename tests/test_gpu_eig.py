"""Eigenvalues without cuSOLVER (csrc/eig_tridiag.cuh): shared-memory
Householder tridiagonalisation (one CTA up to m = 160, a co-resident grid
exchanging one column step at a time through L2 above) + Sturm bisection,
the path of the eager eigen_spectrum and of the eigen route's rank decision
(mset.cpp:153-163) for m <= 2048.
Checked against LAPACK (numpy.linalg.eigvalsh) to 1e-12 of max|lambda| --
the reference's own spectrum pin is 1e-10 (test_mset.cpp:163-199) -- on
random symmetric matrices of awkward sizes, rank-deficient Gram matrices
(duplicate memory vectors, test_mset.cpp:228-234), clustered spectra, and
against the cuSOLVER route of the same library (CSB_EIG_OWN=0; the own
path is the default up to m = 2048)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def p():
    import torch  # noqa: F401
    import paper_2003_08011_b200 as p
    p.context(0)
    return p


@pytest.fixture(autouse=True)
def own_path(monkeypatch):
    # the own solver (the default up to m = 2048; pinned here against a
    # leftover CSB_EIG_OWN=0 in the environment)
    monkeypatch.setenv("CSB_EIG_OWN", "1")


def _err(w, want):
    return float(np.abs(np.asarray(w) - want).max() / max(np.abs(want).max(), 1e-300))


@pytest.mark.parametrize("m", [1, 2, 3, 5, 17, 33, 100, 127, 129, 161, 256, 257, 320, 321, 513, 1000, 1025, 2047,
                               2048])
def test_random_symmetric(p, m):
    rng = np.random.default_rng(m)
    A = rng.standard_normal((m, m))
    A = np.asfortranarray(A + A.T)
    w = p.symmetric_eigvals(A)
    assert (np.diff(w) >= 0).all()
    assert _err(w, np.linalg.eigvalsh(A)) <= 1e-12


@pytest.mark.parametrize("m,dups", [(300, 40), (1000, 7)])
def test_rank_deficient_gram(p, m, dups):
    """Gram matrix of memory vectors with duplicates: exact zero eigenvalues
    (rank < m) must come out at the 1e-12 lambda_max level, like LAPACK."""
    rng = np.random.default_rng(7)
    n = 20
    D = rng.standard_normal((n, m - dups))
    D = np.hstack([D, D[:, :dups]])
    d2 = ((D[:, :, None] - D[:, None, :]) ** 2).sum(0)
    G = np.asfortranarray(1.0 / (1.0 + np.sqrt(d2) / np.sqrt(n)))
    w = p.symmetric_eigvals(G)
    want = np.linalg.eigvalsh(G)
    assert _err(w, want) <= 1e-12
    cut = 1e-10 * want[-1]
    assert (w > cut).sum() == (want > cut).sum() == m - dups  # the rank decision of mset.cpp:156-163


def test_clustered_spectrum(p):
    m = 700
    rng = np.random.default_rng(3)
    Q, _ = np.linalg.qr(rng.standard_normal((m, m)))
    lam = np.concatenate([np.full(300, 1.0), np.full(300, 1.0 + 1e-9), np.linspace(2, 5, 100)])
    A = np.asfortranarray((Q * lam) @ Q.T)
    A = np.asfortranarray(0.5 * (A + A.T))
    assert _err(p.symmetric_eigvals(A), np.linalg.eigvalsh(A)) <= 1e-12


def test_matches_cusolver_route(p, monkeypatch):
    rng = np.random.default_rng(11)
    A = rng.standard_normal((600, 600))
    A = np.asfortranarray(A @ A.T)
    own = p.symmetric_eigvals(A)
    monkeypatch.setenv("CSB_EIG_OWN", "0")
    lib = p.symmetric_eigvals(A)
    assert _err(own, lib) <= 1e-12


@pytest.mark.parametrize("m", [300, 1000])
def test_deterministic(p, m):
    """The grid's reductions have a fixed order (row sums by a fixed
    butterfly, the CTA partials of p^T v summed in CTA order): repeated calls
    are bitwise equal."""
    rng = np.random.default_rng(5)
    A = rng.standard_normal((m, m))
    A = np.asfortranarray(A @ A.T)
    w0 = p.symmetric_eigvals(A)
    for _ in range(3):
        assert np.array_equal(p.symmetric_eigvals(A), w0)


@pytest.mark.parametrize("rows", ["2", "3", "16"])
def test_grid_shapes(p, monkeypatch, rows):
    """Rows per CTA (hence the number of co-resident CTAs, up to one per SM)
    do not change the numbers beyond rounding."""
    monkeypatch.setenv("CSB_EIG_GRID_ROWS", rows)
    m = 145 * int(rows) if rows != "16" else 777  # up to 145 CTAs
    rng = np.random.default_rng(int(rows))
    A = rng.standard_normal((m, m))
    A = np.asfortranarray(A + A.T)
    assert _err(p.symmetric_eigvals(A), np.linalg.eigvalsh(A)) <= 1e-12


@pytest.mark.parametrize("kind", ["diagonal", "tridiagonal", "zero"])
def test_already_reduced_columns(p, kind):
    """Columns with nothing below the subdiagonal give tau = 0 (H = I); the
    grid still runs the column exchange for them (p = 0, w = 0)."""
    m = 400
    rng = np.random.default_rng(9)
    if kind == "diagonal":
        A = np.diag(rng.standard_normal(m))
    elif kind == "tridiagonal":
        e = rng.standard_normal(m - 1)
        A = np.diag(rng.standard_normal(m)) + np.diag(e, 1) + np.diag(e, -1)
    else:
        A = np.zeros((m, m))
    A = np.asfortranarray(A)
    want = np.linalg.eigvalsh(A)
    w = p.symmetric_eigvals(A)
    assert float(np.abs(w - want).max()) <= 1e-12 * max(np.abs(want).max(), 1.0)


@pytest.mark.parametrize("m", [321, 700])
def test_grid_then_one_cta_tail(p, monkeypatch, m):
    """Above m = 320 the grid reduces all but the last 160 columns and the
    one-CTA kernel finishes the trailing block; the same numbers (to
    rounding) as the grid alone (CSB_EIG_NO_TAIL=1)."""
    rng = np.random.default_rng(m)
    A = rng.standard_normal((m, m))
    A = np.asfortranarray(A @ A.T)
    want = np.linalg.eigvalsh(A)
    tail = p.symmetric_eigvals(A)
    monkeypatch.setenv("CSB_EIG_NO_TAIL", "1")
    grid = p.symmetric_eigvals(A)
    assert _err(tail, want) <= 1e-12 and _err(grid, want) <= 1e-12 and _err(tail, grid) <= 1e-12


def test_above_own_range_uses_syevd(p):
    m = 2049
    rng = np.random.default_rng(1)
    A = rng.standard_normal((m, m))
    A = np.asfortranarray(A + A.T)
    assert _err(p.symmetric_eigvals(A), np.linalg.eigvalsh(A)) <= 1e-12


def test_not_symmetric_is_shape_error(p):
    from paper_2003_08011_b200.errors import ShapeError
    A = np.eye(10)
    A[0, 1] = 1.0
    with pytest.raises(ShapeError):
        p.symmetric_eigvals(A)


@pytest.mark.parametrize("m", [2, 40, 100, 160, 200, 500, 1000])
def test_default_path_matches_cusolver(p, monkeypatch, m):
    """The own reduction (one CTA up to 160, the grid above) is the DEFAULT
    eigenvalues-only path (faster than syevd there); CSB_EIG_OWN=0 forces
    syevd."""
    rng = np.random.default_rng(100 + m)
    A = rng.standard_normal((m, m))
    A = np.asfortranarray(A @ A.T + np.eye(m))
    monkeypatch.delenv("CSB_EIG_OWN")
    own = p.symmetric_eigvals(A)
    monkeypatch.setenv("CSB_EIG_OWN", "0")
    lib = p.symmetric_eigvals(A)
    assert _err(own, lib) <= 1e-12 and _err(own, np.linalg.eigvalsh(A)) <= 1e-12
