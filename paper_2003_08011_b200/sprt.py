"""SPRT alarm flags on residual streams (north_star; not in the reference).

The reference stops at residuals (SPEC.md:14 and :190 exclude anomaly
decision logic), so the definition here is this project's: per signal, two
one-sided Wald tests for a mean shift of +-M against N(0, sigma^2), reset on
either decision, computed on the GPU (csrc/sprt.cuh) bit-identically to the
sequential CPU checker oracle/cstress_oracle.c:or_sprt.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from ._lib import check, f64, ptr_d
from .mset import BackendId, _ctx


def sprt_params(sigma, k: float = 3.0, alpha: float = 1e-3, beta: float = 1e-3):
    """c = M / sigma^2, h = M / 2 with M = k sigma (per signal), and the Wald
    thresholds A = ln(beta / (1 - alpha)), B = ln((1 - beta) / alpha)."""
    sigma = np.asarray(sigma, dtype=np.float64)
    if not (np.all(np.isfinite(sigma)) and np.all(sigma > 0)):
        raise ValueError("sprt: sigma must be finite and > 0")
    if not (0 < alpha < 1 and 0 < beta < 1):
        raise ValueError("sprt: alpha and beta must lie in (0, 1)")
    M = k * sigma
    return M / (sigma * sigma), M / 2.0, math.log(beta / (1.0 - alpha)), math.log((1.0 - beta) / alpha)


def residual_sigma(residuals) -> np.ndarray:
    """Population standard deviation per signal of a residual matrix (the
    H0 noise level, e.g. from estimating the training data)."""
    r = np.asarray(residuals, dtype=np.float64)
    return r.std(axis=0)


@dataclass
class SprtDetector:
    """Streaming detector: state (lambda per signal and test) carries across
    update() calls, so feeding a stream in pieces gives the flags of one call."""
    sigma: np.ndarray
    k: float = 3.0
    alpha: float = 1e-3
    beta: float = 1e-3
    backend: BackendId = field(default_factory=BackendId)
    state: Optional[np.ndarray] = None

    def __post_init__(self):
        self.c, self.h, self.A, self.B = sprt_params(self.sigma, self.k, self.alpha, self.beta)
        self.c = np.ascontiguousarray(self.c)
        self.h = np.ascontiguousarray(self.h)
        n = self.c.shape[0]
        if self.state is None:
            self.state = np.zeros((n, 2))
        self.state = np.ascontiguousarray(self.state, dtype=np.float64).reshape(n, 2)

    def update(self, residuals):
        """Host FP64 residuals (N x n) -> (flags N x n uint8, counts (n, 2))."""
        r = f64(residuals)
        N, n = r.shape
        flags = np.zeros((N, n), dtype=np.uint8, order="F")
        counts = np.zeros((n, 2), dtype=np.int64)
        check(_lib.lib().cs_sprt(_ctx(self.backend).handle, ptr_d(r), N, n, ptr_d(self.c), ptr_d(self.h),
                                 self.A, self.B, ptr_d(self.state),
                                 flags.ctypes.data_as(C.POINTER(C.c_uint8)), _lib.ptr_i64(counts)))
        return flags, counts

    def update_device(self, residuals, stream=None):
        """Device residuals (torch, N x n column-major, float32/float64) ->
        device flags (torch uint8, N x n column-major) and host counts."""
        import torch
        N, n = residuals.shape
        if residuals.stride(0) != 1:
            raise ValueError("sprt: residuals must be column-major (stride(0) == 1)")
        ld = residuals.stride(1) if n > 1 else N
        dtype = {torch.float64: 0, torch.float32: 1}[residuals.dtype]
        flags = torch.empty((n, N), dtype=torch.uint8, device=residuals.device).T
        counts = np.zeros((n, 2), dtype=np.int64)
        ctx = _ctx(self.backend)
        st = stream if stream is not None else torch.cuda.current_stream(residuals.device)
        ctx.set_stream(st.cuda_stream)
        try:
            check(_lib.lib().cs_sprt_device(ctx.handle, C.c_void_p(residuals.data_ptr()), dtype, N, n, ld,
                                            ptr_d(self.c), ptr_d(self.h), self.A, self.B, ptr_d(self.state),
                                            C.c_void_p(flags.data_ptr()), _lib.ptr_i64(counts)))
        finally:
            ctx.set_stream(None)
        return flags, counts
