"""The reference's host backends ("reference", "optimized") as a plug-in for
the sweep -- TEST / BASELINE INFRASTRUCTURE ONLY.

The B200 library never computes on the CPU.  To put CPU cells in the same
CostSurface as the b200 cells (the reference times every backend of a
replicate inside one run_cell, /root/reference/proj/src/sweep.cpp:206-227,
and `speedup` divides their medians, surfaces.cpp:100-145), the benchmark's
baseline leg and the tests register this adapter over the CPU oracle with
``paper_2003_08011_b200.estimator.register_host_backend``.
"""
from __future__ import annotations

from . import oracle as o


class OracleHostBackend:
    """train / estimate of the restated reference (mset.cpp:139-199) with the
    backend's own loop nests (backends.cpp:129-293)."""

    def _args(self, backend):
        if backend.kind == "reference":
            return o.REFERENCE, 64, 1
        return o.OPTIMIZED, backend.tile_size, backend.worker_count

    def train(self, X, m, kernel, backend):
        b, tile, workers = self._args(backend)
        h = 0.0 if kernel.bandwidth is None else float(kernel.bandwidth)
        return o.train(X, m, int(kernel.kind), h, b, tile, workers)

    def estimate(self, model, obs, backend):
        b, tile, workers = self._args(backend)
        return o.estimate(model, obs, b, tile, workers)


def register():
    """Register the oracle for both host kinds; returns the adapter."""
    from paper_2003_08011_b200.estimator import register_host_backend
    impl = OracleHostBackend()
    register_host_backend("reference", impl)
    register_host_backend("optimized", impl)
    return impl


def unregister():
    from paper_2003_08011_b200.estimator import unregister_host_backend
    unregister_host_backend("reference")
    unregister_host_backend("optimized")
