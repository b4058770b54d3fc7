"""Host-side mirror of the reference MSET2 interface for the B200 backend.

Mirrors /root/reference/proj/include/containerstress/{kernels,backends,mset}.hpp:
same names, argument meaning and error behaviour, so the parity tests read
like the reference's own tests.  Every compute call goes through the C-ABI
(include/cstress_b200.h) into libcstress_b200.so; nothing here computes on
the CPU.

Layouts follow the reference (types.hpp:7-15): column-major FP64;
signal matrices are observations x signals; memory matrices are
signals x memory vectors.
"""
from __future__ import annotations

import ctypes as C
import math
import re
import threading
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Optional

import numpy as np

from . import _lib
from ._lib import check, f64, ptr_d, ptr_i64
from .errors import ConfigError, ShapeError

# ------------------------------------------------------------------ kernels
class KernelKind(IntEnum):
    """kernels.hpp:12"""
    inverse_distance = 0
    gaussian = 1


@dataclass
class KernelConfig:
    """kernels.hpp:20-35.  bandwidth None -> sqrt(n_signals) at training."""
    kind: KernelKind = KernelKind.inverse_distance
    bandwidth: Optional[float] = None

    def validate(self) -> None:
        if self.bandwidth is not None and not self.bandwidth > 0.0:
            raise ConfigError("kernel bandwidth must be > 0")

    def resolved(self, n_signals: int) -> "KernelConfig":
        return KernelConfig(self.kind, self.bandwidth if self.bandwidth is not None
                            else math.sqrt(float(n_signals)))

    def _h(self) -> float:
        self.validate()
        return float(self.bandwidth) if self.bandwidth is not None else 0.0


PRECISIONS = {"fp64": 0, "fp32": 1}


# ----------------------------------------------------------------- backends
@dataclass(frozen=True)
class BackendId:
    """backends.hpp:14-33 plus the B200 kind this framework implements.

    ``precision`` selects the surveillance arithmetic: ``fp64`` reproduces
    the reference's association and summation order bit-for-bit;
    ``fp32`` runs the fused tcgen05 3xFP16 kernel (tolerance 1e-3).
    """
    kind: str = "b200"
    device: int = 0
    precision: str = "fp64"
    # the reference's host kinds ("reference" / "optimized", backends.hpp:14-33)
    # exist so that CPU and GPU cells share one CostSurface; this library does
    # not compute them -- see register_host_backend
    worker_count: int = 1
    tile_size: int = 64

    def validate(self) -> None:
        if self.kind in HOST_KINDS:  # backends.cpp:86-92
            if self.kind == "optimized":
                if self.worker_count < 1:
                    raise ConfigError("backend worker_count must be >= 1")
                if self.tile_size < 8 or self.tile_size > 1024:
                    raise ConfigError("backend tile_size must lie in [8, 1024]")
            return
        if self.kind != "b200":
            raise ConfigError(f"unknown backend id: {self.kind}")
        if self.device < 0:
            raise ConfigError("backend device must be >= 0")
        if self.precision not in PRECISIONS:
            raise ConfigError(f"unknown precision: {self.precision}")

    @property
    def is_host(self) -> bool:
        return self.kind in HOST_KINDS

    def label(self) -> str:
        if self.kind == "reference":  # backends.cpp:94-99
            return "reference"
        if self.kind == "optimized":
            return f"optimized[tile={self.tile_size}/workers={self.worker_count}]"
        return f"b200[device={self.device}/precision={self.precision}]"

    @staticmethod
    def reference() -> "BackendId":
        return BackendId("reference")

    @staticmethod
    def optimized(workers: int = 0, tile: int = 64) -> "BackendId":
        import os
        b = BackendId("optimized", worker_count=workers or (os.cpu_count() or 1), tile_size=tile)
        b.validate()
        return b

    @staticmethod
    def parse(token: str) -> "BackendId":
        if token == "b200":
            return BackendId()
        if token == "reference":  # backends.cpp:101-111
            return BackendId.reference()
        if token == "optimized":
            return BackendId.optimized()
        m = re.fullmatch(r"optimized\[tile=(-?\d+)/workers=(-?\d+)\]", token)
        if m:
            return BackendId.optimized(int(m.group(2)), int(m.group(1)))
        m = re.fullmatch(r"b200\[device=(\d+)/precision=(fp32|fp64)\]", token)
        if m:
            return BackendId("b200", int(m.group(1)), m.group(2))
        raise ConfigError("unknown backend id: " + token)


HOST_KINDS = ("reference", "optimized")


# ----------------------------------------------------------------- contexts
class Context:
    """One cs_ctx: device + stream + cuSOLVER handle + workspace."""

    def __init__(self, device: int = 0):
        self.device = device
        h = C.c_void_p()
        check(_lib.lib().cs_ctx_create(device, C.byref(h)))
        self.handle = h

    def describe(self) -> str:
        buf = C.create_string_buffer(512)
        check(_lib.lib().cs_ctx_describe(self.handle, buf, 512))
        return buf.value.decode()

    def set_stream(self, stream_ptr: int | None) -> None:
        """stream_ptr: a cudaStream_t value (0 = legacy default stream);
        None restores the context's own stream."""
        if stream_ptr is None:
            check(_lib.lib().cs_ctx_reset_stream(self.handle))
        else:
            check(_lib.lib().cs_ctx_set_stream(self.handle, C.c_void_p(stream_ptr)))

    def synchronize(self) -> None:
        check(_lib.lib().cs_ctx_synchronize(self.handle))

    def __del__(self):
        try:
            if self.handle:
                _lib.lib().cs_ctx_destroy(self.handle)
        except Exception:
            pass


_contexts: dict = {}
_ctx_lock = threading.Lock()


def context(device: int = 0) -> Context:
    key = (threading.get_ident(), device)
    with _ctx_lock:
        if key not in _contexts:
            _contexts[key] = Context(device)
        return _contexts[key]


def _ctx(backend: BackendId) -> Context:
    backend.validate()
    if backend.is_host:
        raise ConfigError(f"backend {backend.label()} is a host CPU backend: this library computes only on "
                          "the B200 (route host backends through estimator.register_host_backend)")
    return context(backend.device)


@dataclass
class BackendCapabilities:
    """backends.hpp:35-41"""
    id: BackendId
    deterministic_summation: bool = True
    description: str = ""


def capabilities(backend: BackendId) -> BackendCapabilities:
    backend.validate()
    if backend.kind == "reference":  # backends.cpp:113-127
        return BackendCapabilities(backend, True, "scalar triple loop, left-to-right accumulation")
    if backend.kind == "optimized":
        return BackendCapabilities(backend, True, f"tiled ({backend.tile_size}x{backend.tile_size}) multi-threaded "
                                   f"({backend.worker_count} workers), depth-blocked strip accumulation")
    return BackendCapabilities(backend, True, _ctx(backend).describe())


# ------------------------------------------------------------ per-op entries
def sim_matrix(A, B, cfg: KernelConfig = KernelConfig(), backend: BackendId = BackendId()):
    """backends.hpp:43-58 -- entry (i, j) = kernel(col i of A, col j of B)."""
    A, B = f64(A), f64(B)
    if A.shape[0] != B.shape[0]:
        raise ShapeError(f"sim_matrix: row counts differ ({A.shape[0]} vs {B.shape[0]})")
    n, p = A.shape
    q = B.shape[1]
    out = np.empty((p, q), order="F")
    check(_lib.lib().cs_sim_matrix(_ctx(backend).handle, ptr_d(A), ptr_d(B), n, p, q,
                                   int(cfg.kind), cfg._h(), ptr_d(out)))
    return out


similarity_matrix = sim_matrix  # mset.hpp:65-70


def matmul(A, B, backend: BackendId = BackendId()):
    """backends.hpp:60-61"""
    A, B = f64(A), f64(B)
    if A.shape[1] != B.shape[0]:
        raise ShapeError(f"matmul: inner dimensions differ ({A.shape[1]} vs {B.shape[0]})")
    out = np.empty((A.shape[0], B.shape[1]), order="F")
    check(_lib.lib().cs_matmul(_ctx(backend).handle, ptr_d(A), ptr_d(B), A.shape[0], A.shape[1],
                               B.shape[1], ptr_d(out)))
    return out


def batched_solve(G_pinv, S, backend: BackendId = BackendId()):
    """backends.hpp:63-65 (== matmul(G_pinv, S))"""
    G_pinv, S = f64(G_pinv), f64(S)
    if G_pinv.shape[1] != S.shape[0]:
        raise ShapeError("batched_solve: G_pinv columns must match S rows")
    out = np.empty((G_pinv.shape[0], S.shape[1]), order="F")
    check(_lib.lib().cs_batched_solve(_ctx(backend).handle, ptr_d(G_pinv), ptr_d(S),
                                      G_pinv.shape[0], S.shape[1], ptr_d(out)))
    return out


@dataclass
class SymmetricEig:
    eigenvalues: np.ndarray
    eigenvectors: np.ndarray


def symmetric_eig(G, backend: BackendId = BackendId()) -> SymmetricEig:
    """mset.hpp:34-38"""
    G = f64(G)
    if G.ndim != 2 or G.shape[0] != G.shape[1]:
        raise ShapeError("symmetric_eig: matrix is not square")
    m = G.shape[0]
    w = np.empty(m)
    V = np.empty((m, m), order="F")
    check(_lib.lib().cs_symmetric_eig(_ctx(backend).handle, ptr_d(G), m, ptr_d(w), ptr_d(V)))
    return SymmetricEig(w, V)


def symmetric_eigvals(G, backend: BackendId = BackendId()) -> np.ndarray:
    """The eigenvalues (ascending) of symmetric_eig (mset.hpp:34-38) without
    the vectors (cs_symmetric_eigvals): for m <= 2048 the library's own
    shared-memory tridiagonalisation + bisection (CSB_EIG_OWN=0: cuSOLVER
    syevd), above it syevd."""
    G = f64(G)
    if G.ndim != 2 or G.shape[0] != G.shape[1]:
        raise ShapeError("symmetric_eig: matrix is not square")
    m = G.shape[0]
    w = np.empty(m)
    check(_lib.lib().cs_symmetric_eigvals(_ctx(backend).handle, ptr_d(G), m, ptr_d(w)))
    return w


@dataclass
class MemoryMatrix:
    """mset.hpp:21-27"""
    D: np.ndarray
    source_indices: list

    def n_signals(self):
        return self.D.shape[0]

    def n_memory(self):
        return self.D.shape[1]


def _signal_data(x):
    return f64(getattr(x, "data", x))


def select_memory_vectors(training, m: int, backend: BackendId = BackendId()) -> MemoryMatrix:
    """mset.hpp:40-43 / mset.cpp:72-137 (bit-exact indices)."""
    X = _signal_data(training)
    N, n = X.shape
    idx = np.empty(m, dtype=np.int64)
    D = np.empty((n, m), order="F")
    check(_lib.lib().cs_select_memory_vectors(_ctx(backend).handle, ptr_d(X), N, n, m,
                                              ptr_i64(idx), ptr_d(D)))
    return MemoryMatrix(D, idx.tolist())


# ------------------------------------------------------------ train/estimate
class TrainedModel:
    """Device-resident TrainedModel (mset.hpp:46-57); immutable after training."""

    def __init__(self, handle: C.c_void_p, backend: BackendId):
        self.handle = handle
        self.backend = backend
        n, m, r, kind, prec = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int(), C.c_int()
        h = C.c_double()
        check(_lib.lib().cs_model_info(handle, C.byref(n), C.byref(m), C.byref(r), C.byref(kind),
                                       C.byref(h), C.byref(prec)))
        self._n, self._m, self.rank = n.value, m.value, r.value
        self.kernel = KernelConfig(KernelKind(kind.value), h.value)
        self.precision = prec.value
        self._export = None

    def n_signals(self):
        return self._n

    def n_memory(self):
        return self._m

    def export(self) -> dict:
        if self._export is None:
            n, m = self._n, self._m
            idx = np.empty(m, dtype=np.int64)
            D = np.empty((n, m), order="F")
            pinv = np.empty((m, m), order="F")
            spec = np.empty(m)
            scale = np.empty(n)
            check(_lib.lib().cs_model_export(self.handle, ptr_i64(idx), ptr_d(D), ptr_d(pinv),
                                             ptr_d(spec), ptr_d(scale)))
            self._export = dict(source_indices=idx, D=D, gram_pinv=pinv, eigen_spectrum=spec,
                                signal_scale=scale)
        return self._export

    @property
    def memory(self) -> MemoryMatrix:
        e = self.export()
        return MemoryMatrix(e["D"], e["source_indices"].tolist())

    @property
    def gram_pinv(self):
        return self.export()["gram_pinv"]

    @property
    def eigen_spectrum(self):
        return self.export()["eigen_spectrum"]

    @property
    def signal_scale(self):
        return self.export()["signal_scale"]

    @property
    def memory_normalized(self):
        e = self.export()
        return e["D"] / e["signal_scale"][:, None]

    def __del__(self):
        try:
            if self.handle:
                _lib.lib().cs_model_destroy(self.handle)
        except Exception:
            pass


def train(training, m: int, cfg: KernelConfig = KernelConfig(),
          backend: BackendId = BackendId()) -> TrainedModel:
    """mset.hpp:72-77 / mset.cpp:139-172."""
    X = _signal_data(training)
    N, n = X.shape
    h = C.c_void_p()
    check(_lib.lib().cs_mset_train(_ctx(backend).handle, ptr_d(X), N, n, m, int(cfg.kind),
                                   cfg._h(), PRECISIONS[backend.precision], C.byref(h)))
    return TrainedModel(h, backend)


def train_device(training, m: int, cfg: KernelConfig = KernelConfig(),
                 backend: BackendId = BackendId()) -> TrainedModel:
    """train on a device-resident float64 torch tensor (N x n column-major,
    i.e. stride(0) == 1 and leading dimension N)."""
    import torch
    if training.dtype != torch.float64 or training.dim() != 2 or training.stride(0) != 1:
        raise ShapeError("train_device: training must be a column-major float64 N x n tensor")
    N, n = training.shape
    if n > 1 and training.stride(1) != N:
        raise ShapeError("train_device: training must be contiguous column-major (ld == N)")
    _check_device(training, backend, "train_device: training")
    ctx = _ctx(backend)
    # the library runs on torch's current stream, so a producer still writing
    # `training` asynchronously on that stream is ordered before the train
    ctx.set_stream(torch.cuda.current_stream(training.device).cuda_stream)
    h = C.c_void_p()
    try:
        check(_lib.lib().cs_mset_train_device(ctx.handle, C.c_void_p(training.data_ptr()), N, n,
                                              m, int(cfg.kind), cfg._h(), PRECISIONS[backend.precision],
                                              C.byref(h)))
    finally:
        ctx.set_stream(None)
    return TrainedModel(h, backend)


def _check_device(t, backend: BackendId, what: str) -> None:
    if not t.is_cuda or t.device.index != backend.device:
        raise ConfigError(f"{what} must be a CUDA tensor on device {backend.device} (got {t.device})")


def import_model(D, signal_scale, gram_pinv, rank, cfg: KernelConfig,
                 backend: BackendId = BackendId(), source_indices=None,
                 eigen_spectrum=None) -> TrainedModel:
    """Host TrainedModel -> device (the load_model path, mset.cpp:269-310)."""
    D, sc, pv = f64(D), f64(signal_scale), f64(gram_pinv)
    n, m = D.shape
    idx = None if source_indices is None else np.ascontiguousarray(source_indices, dtype=np.int64)
    sp = None if eigen_spectrum is None else f64(eigen_spectrum)
    h = C.c_void_p()
    check(_lib.lib().cs_model_import(
        _ctx(backend).handle, n, m, int(cfg.kind), cfg._h(), int(rank),
        ptr_i64(idx) if idx is not None else None, ptr_d(D), ptr_d(pv),
        ptr_d(sp) if sp is not None else None, ptr_d(sc), PRECISIONS[backend.precision],
        C.byref(h)))
    return TrainedModel(h, backend)


def save_model(model: TrainedModel, path: str) -> None:
    """save_model (mset.hpp:85, mset.cpp:229-267): CSM1 binary + .json sidecar."""
    check(_lib.lib().cs_model_save(model.handle, str(path).encode()))


def load_model(path: str, backend: BackendId = BackendId()) -> TrainedModel:
    """load_model (mset.hpp:86, mset.cpp:269-310) onto the backend's device."""
    h = C.c_void_p()
    check(_lib.lib().cs_model_load(_ctx(backend).handle, str(path).encode(), PRECISIONS[backend.precision],
                                   C.byref(h)))
    return TrainedModel(h, backend)


@dataclass
class EstimationResult:
    """mset.hpp:59-62"""
    estimates: np.ndarray
    residuals: np.ndarray


def estimate(model: TrainedModel, observations, backend: Optional[BackendId] = None
             ) -> EstimationResult:
    """mset.hpp:79-82 / mset.cpp:174-199 -- host FP64 in and out."""
    backend = backend or model.backend
    obs = _signal_data(observations)
    N, n = obs.shape
    est = np.empty((N, n), order="F")
    res = np.empty((N, n), order="F")
    check(_lib.lib().cs_mset_estimate(_ctx(backend).handle, model.handle, ptr_d(obs), N, n,
                                      ptr_d(est), ptr_d(res)))
    return EstimationResult(est, res)


def estimate_device(model: TrainedModel, obs, est=None, resid=None, stream=None,
                    backend: Optional[BackendId] = None):
    """Device-resident surveillance on torch CUDA tensors (N x n column-major,
    i.e. tensors whose transpose is contiguous, or 1-D views with ld).

    Asynchronous on ``stream`` (a torch.cuda.Stream, default: current)."""
    import torch
    backend = backend or model.backend
    if obs.dim() != 2 or obs.stride(0) != 1:
        raise ShapeError("estimate_device: observations must be column-major (N x n, stride(0)==1)")
    N, n = obs.shape
    ld = obs.stride(1) if n > 1 else N
    dtype = {torch.float32: 1, torch.float64: 0}.get(obs.dtype)
    if dtype is None:
        raise ConfigError("estimate_device: observations must be float32 or float64")
    _check_device(obs, backend, "estimate_device: observations")
    # outputs are written as N x n values of obs's dtype at obs's leading
    # dimension: anything else would be written out of bounds or transposed
    for name, t in (("estimates", est), ("residuals", resid)):
        if t is None:
            continue
        _check_device(t, backend, f"estimate_device: {name}")
        if t.dtype != obs.dtype or tuple(t.shape) != (N, n) or t.stride(0) != 1 or (n > 1 and t.stride(1) != ld):
            raise ShapeError(f"estimate_device: {name} must match the observations' dtype, shape and "
                             f"column-major strides ({obs.dtype}, {(N, n)}, ld={ld})")
        if t.storage_offset() + (ld * (n - 1) + N if N and n else 0) > t.untyped_storage().nbytes() // t.element_size():
            raise ShapeError(f"estimate_device: {name} storage is smaller than N x ld")
    ctx = _ctx(backend)
    st = stream if stream is not None else torch.cuda.current_stream(obs.device)
    ctx.set_stream(st.cuda_stream)
    try:
        check(_lib.lib().cs_mset_estimate_device(
            ctx.handle, model.handle, C.c_void_p(obs.data_ptr()), dtype, N, n, ld,
            C.c_void_p(est.data_ptr() if est is not None else 0),
            C.c_void_p(resid.data_ptr() if resid is not None else 0)))
    finally:
        ctx.set_stream(None)


# ------------------------------------------------------------- model wire
def pack_model(model: TrainedModel, out=None):
    """The whole device model as one uint8 CUDA tensor on the model's device
    (cs_model_pack_device): what rank 0 broadcasts in the observation-sharded
    C5' path.  `out` may be a preallocated uint8 tensor."""
    import torch
    nbytes = C.c_int64()
    check(_lib.lib().cs_model_wire_size(model.handle, C.byref(nbytes)))
    dev = torch.device("cuda", model.backend.device)
    if out is None:
        out = torch.empty(nbytes.value, dtype=torch.uint8, device=dev)
    if out.dtype != torch.uint8 or not out.is_contiguous() or out.numel() < nbytes.value:
        raise ShapeError("pack_model: out must be a contiguous uint8 tensor of at least the wire size")
    _check_device(out, model.backend, "pack_model: out")
    ctx = _ctx(model.backend)
    ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
    try:
        check(_lib.lib().cs_model_pack_device(ctx.handle, model.handle, C.c_void_p(out.data_ptr()),
                                              out.numel()))
    finally:
        ctx.set_stream(None)
    return out


def unpack_model(wire, backend: BackendId = BackendId()) -> TrainedModel:
    """A model from a wire tensor (cs_model_unpack_device) on the backend's
    device; its estimates are bitwise those of the packed model."""
    import torch
    if wire.dtype != torch.uint8 or not wire.is_contiguous():
        raise ShapeError("unpack_model: wire must be a contiguous uint8 tensor")
    _check_device(wire, backend, "unpack_model: wire")
    ctx = _ctx(backend)
    ctx.set_stream(torch.cuda.current_stream(wire.device).cuda_stream)
    h = C.c_void_p()
    try:
        check(_lib.lib().cs_model_unpack_device(ctx.handle, C.c_void_p(wire.data_ptr()), wire.numel(),
                                                C.byref(h)))
    finally:
        ctx.set_stream(None)
    return TrainedModel(h, backend)
