"""Plugin contract mirror (estimator.hpp:10-59, estimator.cpp:17-69).

``MsetAlgorithm`` routes whole train / estimate calls to the C-ABI for the
``b200`` backend kind; the returned model is an opaque device-resident
``PrognosticModel``.  ``MeanPredictor`` is the reference's trivial baseline
(estimator.hpp:45-56) kept for the pluggability contract.
"""
from __future__ import annotations

import numpy as np

from . import mset
from .errors import ConfigError, ShapeError
from .mset import BackendId, EstimationResult, KernelConfig


class PrognosticModel:
    """estimator.hpp:11-14 (opaque)."""


class MsetModel(PrognosticModel):
    def __init__(self, model: mset.TrainedModel):
        self.model = model


class HostMsetModel(PrognosticModel):
    """A model trained by a registered host (CPU) backend."""

    def __init__(self, model, kind: str):
        self.model = model
        self.kind = kind


class MeanModel(PrognosticModel):
    def __init__(self, means):
        self.means = means


def _as(model, cls, algo):
    # estimator.cpp:17-23
    if not isinstance(model, cls):
        raise ConfigError("model was not trained by algorithm " + algo)
    return model


class PrognosticAlgorithm:
    """estimator.hpp:18-29"""

    def name(self) -> str:
        raise NotImplementedError

    def train(self, training, n_memory: int, kernel: KernelConfig, backend: BackendId):
        raise NotImplementedError

    def estimate(self, model, observations, backend: BackendId) -> EstimationResult:
        raise NotImplementedError


# Host (CPU) implementations of the reference's own backend kinds
# ("reference", "optimized"; backends.hpp:14-33).  The B200 library never
# computes on the CPU; a host implementation is registered by whoever wants
# CPU cells in the same CostSurface as the b200 cells (the reference runs
# every backend of a replicate inside one run_cell, sweep.cpp:206-227) --
# here the benchmark's baseline leg and the tests, which register the CPU
# oracle.  An implementation provides
#   train(X, m, kernel: KernelConfig, backend) -> opaque host model
#   estimate(model, observations, backend) -> (estimates, residuals)
_HOST_BACKENDS: dict = {}


def register_host_backend(kind: str, impl) -> None:
    if kind not in mset.HOST_KINDS:
        raise ConfigError("unknown host backend kind: " + kind)
    _HOST_BACKENDS[kind] = impl


def unregister_host_backend(kind: str) -> None:
    _HOST_BACKENDS.pop(kind, None)


def host_backend(backend: BackendId):
    backend.validate()
    impl = _HOST_BACKENDS.get(backend.kind)
    if impl is None:
        raise ConfigError(f"backend {backend.label()} has no host implementation registered "
                          "(this library computes only on the B200)")
    return impl


class MsetAlgorithm(PrognosticAlgorithm):
    def name(self):
        return "mset2"

    def train(self, training, n_memory, kernel=KernelConfig(), backend=BackendId()):
        if backend.is_host:
            X = np.asfortranarray(np.asarray(getattr(training, "data", training), dtype=np.float64))
            return HostMsetModel(host_backend(backend).train(X, n_memory, kernel, backend), backend.kind)
        return MsetModel(mset.train(training, n_memory, kernel, backend))

    def estimate(self, model, observations, backend=BackendId()):
        if backend.is_host:
            impl = host_backend(backend)
            hm = _as(model, HostMsetModel, "mset2")
            obs = np.asfortranarray(np.asarray(getattr(observations, "data", observations), dtype=np.float64))
            est, res = impl.estimate(hm.model, obs, backend)
            return EstimationResult(est, res)
        return mset.estimate(_as(model, MsetModel, "mset2").model, observations, backend)


class MeanPredictor(PrognosticAlgorithm):
    def name(self):
        return "mean"

    def train(self, training, n_memory, kernel=KernelConfig(), backend=BackendId()):
        X = np.asarray(getattr(training, "data", training))
        return MeanModel(X.mean(axis=0))

    def estimate(self, model, observations, backend=BackendId()):
        means = _as(model, MeanModel, "mean").means
        X = np.asarray(getattr(observations, "data", observations))
        if X.shape[1] != means.shape[0]:
            raise ShapeError("mean predictor: signal count mismatch")
        est = np.asfortranarray(np.broadcast_to(means, X.shape))
        return EstimationResult(est, np.asfortranarray(X - est))


_REGISTRY = {"mset2": MsetAlgorithm(), "mean": MeanPredictor()}


def algorithm_by_name(name: str) -> PrognosticAlgorithm:
    """estimator.cpp:63-69"""
    if name not in _REGISTRY:
        raise ConfigError("unknown estimator: " + name)
    return _REGISTRY[name]
