#!/usr/bin/env python
"""Generate the large-config golden fixtures (tests/golden/mset_c3.npz,
tests/golden/mset_c5.npz) from the CPU oracle -- TEST INFRASTRUCTURE.

The oracle's own `or_train` uses a hand-written tred2/tql2 eigensolver, which
is pinned by the reference's known-answer and relational tests
(tests/test_oracle_mset.py) but takes hours single-threaded at m = 8000.  At
these sizes the train below restates mset.cpp:139-170 step by step with the
oracle's pinned pieces and LAPACK's `dsyevd` (scipy.linalg.eigh, driver
"evd") in place of Eigen's SelfAdjointEigenSolver (LAPACK dsyevd
is the stronger-than-Eigen substitute; the contract it must meet is
mset.hpp:34-38: ascending eigenvalues, orthonormal vectors):

  select_memory_vectors    mset.cpp:142         or_select_memory_vectors
  resolved bandwidth       mset.cpp:143         h = sqrt(n) (kernels.hpp:30-34)
  per_signal_scale         mset.cpp:145         or_per_signal_scale
  memory_normalized        mset.cpp:147-149     D / scale, row-wise
  gram = sim_matrix(Dn,Dn) mset.cpp:151-152     or_sim_matrix_optimized (tile 64, all cores)
  symmetric_eig            mset.cpp:153         LAPACK dsyevd
  cutoff, rank             mset.cpp:156-163     lambda > 1e-10 * lambda_max
  whitened, gram_pinv      mset.cpp:165-170     W = V_k / sqrt(lambda_k); or_matmul_optimized(W, W^T)
  estimate                 mset.cpp:174-199     or_estimate (optimized backend)

Inputs are the sweep's own data recipe: training rows = 4 m synthesized from
derive_seed(cell_data_seed(20260810, n, N, m, 0), {0}) with the demo
template (docs/demo_sweep.json:12-18), surveillance sample rows from
derive_seed(base, {1}) (sweep.cpp:153-166).  The fixtures hold what a GPU
test needs to check a B200 train at full size without the 128 MB - 512 MB
matrices: source indices, scale, spectrum, rank, G+ applied to four seeded
probe vectors, the estimates of a surveillance sample, and checksums of the
training rows (so a test knows it fed the same bytes).

Usage: python tools/make_golden.py [c3] [c5]     (c3 ~3 min, c5 ~15 min on 8 cores)
"""
from __future__ import annotations

import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as o  # noqa: E402

MASTER = 20260810
TEMPLATE = (0.5, 0.3, 1.0, 0.5, 4.0)  # phi, rho, variance, skew, kurt
PROBE_SEED = 20261017

CONFIGS = {
    # name: (n, N (cell coordinate), m, surveillance sample rows)
    "c3": (1000, 1_000_000, 4000, 128),
    "c5": (4000, 10_000_000, 8000, 32),
}


def train_lapack(X, m, workers):
    import scipy.linalg as sl
    N, n = X.shape
    idx, D = o.select_memory_vectors(X, m)
    h = math.sqrt(n)
    scale = o.per_signal_scale(X)
    Dn = np.asfortranarray(D / scale[:, None])
    t = time.time()
    G = o.sim_matrix_optimized(Dn, Dn, o.INVERSE_DISTANCE, h, 64, workers)
    print(f"  gram {time.time() - t:.1f} s", flush=True)
    t = time.time()
    w, V = sl.eigh(G, driver="evd", overwrite_a=False, check_finite=False)
    print(f"  dsyevd {time.time() - t:.1f} s", flush=True)
    cutoff = 1e-10 * w[m - 1]
    kept = np.nonzero(w > cutoff)[0]
    rank = len(kept)
    W = np.asfortranarray(V[:, kept] / np.sqrt(w[kept])[None, :])
    t = time.time()
    pinv = o.matmul_optimized(W, np.asfortranarray(W.T), 64, workers)
    print(f"  pinv {time.time() - t:.1f} s", flush=True)
    model = o.Model(source_indices=idx, D=D, scale=scale, gram_pinv=pinv, eigen_spectrum=w,
                    rank=rank, h=h, kind=o.INVERSE_DISTANCE)
    return model, G


def checksums(X):
    return np.array([X.sum(), (X * X).sum(), X[::997, ::13].sum()])


def make(name, workers):
    n, Ncell, m, ns = CONFIGS[name]
    base = o.cell_data_seed(MASTER, n, Ncell, m, 0)
    t = time.time()
    X = o.synthesize_uniform(n, 4 * m, *TEMPLATE, o.derive_seed(base, [0]))
    obs = o.synthesize_uniform(n, ns, *TEMPLATE, o.derive_seed(base, [1]))
    print(f"{name}: synth {time.time() - t:.1f} s", flush=True)
    model, G = train_lapack(X, m, workers)
    probes = np.random.default_rng(PROBE_SEED).standard_normal((m, 4))
    pinv_probes = model.gram_pinv @ probes
    t = time.time()
    est, res = o.estimate(model, obs, o.OPTIMIZED, 64, workers)
    print(f"  estimate {time.time() - t:.1f} s; rank {model.rank}/{m}, "
          f"lambda {model.eigen_spectrum[0]:.3e} .. {model.eigen_spectrum[-1]:.3e}", flush=True)
    out = os.path.join(ROOT, "tests", "golden", f"mset_{name}.npz")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    np.savez_compressed(
        out, n=n, N_cell=Ncell, m=m, master_seed=MASTER, template=np.array(TEMPLATE),
        train_seed=np.uint64(o.derive_seed(base, [0])), obs_seed=np.uint64(o.derive_seed(base, [1])),
        sample_rows=ns, h=model.h, rank=model.rank, source_indices=model.source_indices,
        scale=model.scale, spectrum=model.eigen_spectrum, probe_seed=PROBE_SEED,
        pinv_probes=pinv_probes, pinv_diag=np.diag(model.gram_pinv).copy(),
        gram_diag_check=np.array([np.abs(np.diag(G) - 1.0).max()]),
        est=est, train_checksums=checksums(X), obs_checksums=checksums(obs),
        generator="tools/make_golden.py (oracle pieces + LAPACK dsyevd)")
    print(f"  wrote {out} ({os.path.getsize(out) / 1e6:.2f} MB)", flush=True)


def main():
    o.build()
    workers = os.cpu_count() or 1
    names = [a for a in sys.argv[1:] if a in CONFIGS] or list(CONFIGS)
    for nm in names:
        make(nm, workers)


if __name__ == "__main__":
    main()
