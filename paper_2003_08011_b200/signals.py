"""Data feed: SignalSpec / SignalMatrix / synthesize for uniform specs.

Mirrors signals.hpp:23-51 and synthesize (signals.cpp:205-254) through the
C-ABI (``cs_synthesize_uniform``).  Untimed in the reference harness
(sweep.cpp:207-208).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from ._lib import check, ptr_d


@dataclass
class SignalSpec:
    """SignalSpec::uniform (signals.cpp:51-65): scalar targets broadcast to
    every channel, uniform off-diagonal correlation rho."""
    n_signals: int
    n_observations: int
    ar_coefficient: float = 0.0
    cross_correlation: float = 0.0
    variance: float = 1.0
    skewness: float = 0.0
    kurtosis: float = 3.0
    seed: int = 0

    @staticmethod
    def uniform(n, N, phi, rho, variance, skewness, kurtosis, seed) -> "SignalSpec":
        return SignalSpec(n, N, phi, rho, variance, skewness, kurtosis, seed)


@dataclass
class SignalMatrix:
    """signals.hpp:45-51: rows = observations, columns = signals."""
    data: np.ndarray
    spec: Optional[SignalSpec] = None

    def n_observations(self):
        return self.data.shape[0]

    def n_signals(self):
        return self.data.shape[1]


def synthesize(spec: SignalSpec) -> SignalMatrix:
    out = np.empty((spec.n_observations, spec.n_signals), order="F")
    check(_lib.lib().cs_synthesize_uniform(
        spec.n_signals, spec.n_observations, spec.ar_coefficient, spec.cross_correlation,
        spec.variance, spec.skewness, spec.kurtosis, spec.seed & (2**64 - 1), ptr_d(out)))
    return SignalMatrix(out, spec)


def synthesize_device(spec: SignalSpec, device: int = 0, dtype=None):
    """Same recipe on the GPU; returns an N x n column-major torch tensor on
    cuda:device (tolerance parity with ``synthesize``).  float64 by default;
    ``dtype=torch.float32`` rounds the final FP64 values once in the last
    pass (bit-identical to ``synthesize_device(spec).float()``)."""
    import torch
    from .mset import context
    dev = torch.device("cuda", device)
    ctx = context(device)
    args = (ctx.handle, spec.n_signals, spec.n_observations, spec.ar_coefficient, spec.cross_correlation,
            spec.variance, spec.skewness, spec.kurtosis, spec.seed & (2**64 - 1))
    if dtype is None or dtype == torch.float64:
        out = torch.empty((spec.n_signals, spec.n_observations), dtype=torch.float64, device=dev).T
        check(_lib.lib().cs_synthesize_uniform_device(*args, out.data_ptr()))
        return out
    if dtype != torch.float32:
        raise ValueError("synthesize_device: dtype must be float64 or float32")
    work = torch.empty((spec.n_signals, spec.n_observations), dtype=torch.float64, device=dev)
    out = torch.empty((spec.n_signals, spec.n_observations), dtype=torch.float32, device=dev).T
    check(_lib.lib().cs_synthesize_uniform_device_f32(*args, work.data_ptr(), out.data_ptr()))
    return out


def derive_seed(parent: int, coords) -> int:
    import ctypes as C
    arr = (C.c_uint64 * max(len(coords), 1))(*coords)
    return _lib.lib().cs_derive_seed(parent, arr, len(coords))


def cell_data_seed(master: int, n: int, N: int, m: int, replicate: int) -> int:
    """sweep.cpp:119-126"""
    return _lib.lib().cs_cell_data_seed(master, n, N, m, replicate)
