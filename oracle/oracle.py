"""ctypes view of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this module.  It is the checker the
B200 product is compared against, never part of the product path.

Every function restates the reference (``/root/reference/proj``) at the
file:line given in ``cstress_oracle.c``.  Arrays follow the reference layout:
column-major (Fortran-order) FP64, observations x signals for signal
matrices (``types.hpp:13``, ``signals.hpp:45-51``).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

OK = 0
ERROR_NAMES = {
    1: "Error", 2: "ConstraintViolated", 3: "InsufficientTraining",
    4: "DegenerateModel", 5: "EigFailure", 6: "ShapeError", 7: "ConfigError",
    8: "IoError", 9: "MomentInfeasible", 10: "BadCorrelation",
    11: "TooFewSamples", 12: "EmptyGrid",
}
INVERSE_DISTANCE, GAUSSIAN = 0, 1
REFERENCE, OPTIMIZED = 0, 1


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code
        self.kind = ERROR_NAMES.get(code, "Error")


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        P = C.POINTER
        d, i64, u64, i32 = C.c_double, C.c_int64, C.c_uint64, C.c_int
        pd, pi64, pu64 = P(d), P(i64), P(u64)
        sig = {
            "or_last_error": (C.c_char_p, []),
            "or_splitmix64_mix": (u64, [u64]),
            "or_derive_seed": (u64, [u64, pu64, i32]),
            "or_gaussian_fill": (None, [u64, i64, pd]),
            "or_testrng_matrix": (None, [pu64, i64, i64, d, d, pd]),
            "or_testrng_uniform_int": (i32, [pu64, i32, i32]),
            "or_solve_fleishman": (i32, [d, d, pd]),
            "or_nearest_psd_repair": (i32, [pd, i64, d, pd, pd]),
            "or_synthesize": (i32, [i64, i64, d, pd, pd, pd, pd, u64, pd]),
            "or_synthesize_uniform": (i32, [i64, i64, d, d, d, d, d, u64, pd]),
            "or_kernel_from_d2": (d, [d, i32, d]),
            "or_fnv1a_row": (u64, [pd, i64, i64]),
            "or_count_distinct_rows": (i64, [pd, i64, i64]),
            "or_select_memory_vectors": (i32, [pd, i64, i64, i64, pi64, pd]),
            "or_per_signal_scale": (None, [pd, i64, i64, pd]),
            "or_sim_matrix_reference": (i32, [pd, pd, i64, i64, i64, i32, d, pd]),
            "or_sim_matrix_optimized": (i32, [pd, pd, i64, i64, i64, i32, d, i32, i32, pd]),
            "or_matmul_reference": (i32, [pd, pd, i64, i64, i64, pd]),
            "or_matmul_optimized": (i32, [pd, pd, i64, i64, i64, i32, i32, pd]),
            "or_symmetric_eig": (i32, [pd, i64, pd, pd]),
            "or_jacobi_eig": (None, [pd, i64, pd, pd]),
            "or_train": (i32, [pd, i64, i64, i64, i32, d, i32, i32, i32, pi64, pd,
                               pd, pd, pd, pi64, pd]),
            "or_estimate": (i32, [pd, pd, pd, i64, i64, i64, i32, d, pd, i64, i32,
                                  i32, i32, pd, pd]),
            "or_cell_data_seed": (u64, [u64, i64, i64, i64, i32]),
            "or_sprt": (None, [pd, i64, i64, i64, pd, pd, C.c_double, C.c_double, pd,
                               C.POINTER(C.c_uint8), pi64]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _pd(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _pi64(a):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


def _f64(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _check(code):
    if code != OK:
        raise OracleError(code, lib().or_last_error().decode())


# ----------------------------------------------------------------- rng
def splitmix64_mix(z: int) -> int:
    return lib().or_splitmix64_mix(z)


def derive_seed(parent: int, coords) -> int:
    arr = (C.c_uint64 * max(len(coords), 1))(*coords)
    return lib().or_derive_seed(parent, arr, len(coords))


def gaussian_stream(seed: int, count: int) -> np.ndarray:
    out = np.empty(count)
    lib().or_gaussian_fill(seed, count, _pd(out))
    return out


class TestRng:
    """oracles::TestRng (tests/support/oracles.hpp:173-203)."""

    __test__ = False  # not a pytest class

    def __init__(self, seed: int):
        self.state = C.c_uint64(seed if seed else 1)

    def matrix(self, rows, cols, lo, hi):
        out = np.empty((rows, cols), order="F")
        lib().or_testrng_matrix(C.byref(self.state), rows, cols, lo, hi, _pd(out))
        return out

    def uniform_int(self, lo, hi):
        return lib().or_testrng_uniform_int(C.byref(self.state), lo, hi)


# ------------------------------------------------------------- signals
def solve_fleishman(skew, kurt):
    out = np.empty(4)
    _check(lib().or_solve_fleishman(skew, kurt, _pd(out)))
    return out  # a, b, c, d


def nearest_psd_repair(corr, jitter_cap):
    corr = _f64(corr)
    n = corr.shape[0]
    out = np.empty((n, n), order="F")
    jit = np.zeros(1)
    _check(lib().or_nearest_psd_repair(_pd(corr), n, jitter_cap, _pd(out), _pd(jit)))
    return out, float(jit[0])


def synthesize_uniform(n, N, phi, rho, variance, skew, kurt, seed):
    out = np.empty((N, n), order="F")
    _check(lib().or_synthesize_uniform(n, N, phi, rho, variance, skew, kurt, seed, _pd(out)))
    return out


# ---------------------------------------------------------------- mset
def kernel_from_d2(d2, kind, h):
    return lib().or_kernel_from_d2(d2, kind, h)


def count_distinct_rows(X):
    X = _f64(X)
    return lib().or_count_distinct_rows(_pd(X), X.shape[0], X.shape[1])


def select_memory_vectors(X, m):
    X = _f64(X)
    N, n = X.shape
    idx = np.empty(m, dtype=np.int64)
    D = np.empty((n, m), order="F")
    _check(lib().or_select_memory_vectors(_pd(X), N, n, m, _pi64(idx), _pd(D)))
    return idx, D


def per_signal_scale(X):
    X = _f64(X)
    out = np.empty(X.shape[1])
    lib().or_per_signal_scale(_pd(X), X.shape[0], X.shape[1], _pd(out))
    return out


def sim_matrix_reference(A, B, kind=INVERSE_DISTANCE, h=0.0):
    A, B = _f64(A), _f64(B)
    if A.shape[0] != B.shape[0]:
        raise OracleError(6, "sim_matrix: row counts differ")
    out = np.empty((A.shape[1], B.shape[1]), order="F")
    _check(lib().or_sim_matrix_reference(_pd(A), _pd(B), A.shape[0], A.shape[1],
                                         B.shape[1], kind, h, _pd(out)))
    return out


def sim_matrix_optimized(A, B, kind=INVERSE_DISTANCE, h=0.0, tile=64, workers=1):
    A, B = _f64(A), _f64(B)
    if A.shape[0] != B.shape[0]:
        raise OracleError(6, "sim_matrix: row counts differ")
    out = np.empty((A.shape[1], B.shape[1]), order="F")
    _check(lib().or_sim_matrix_optimized(_pd(A), _pd(B), A.shape[0], A.shape[1],
                                         B.shape[1], kind, h, tile, workers, _pd(out)))
    return out


def matmul_reference(A, B):
    A, B = _f64(A), _f64(B)
    if A.shape[1] != B.shape[0]:
        raise OracleError(6, "matmul: inner dimensions differ")
    out = np.empty((A.shape[0], B.shape[1]), order="F")
    _check(lib().or_matmul_reference(_pd(A), _pd(B), A.shape[0], A.shape[1], B.shape[1], _pd(out)))
    return out


def matmul_optimized(A, B, tile=64, workers=1):
    A, B = _f64(A), _f64(B)
    if A.shape[1] != B.shape[0]:
        raise OracleError(6, "matmul: inner dimensions differ")
    out = np.empty((A.shape[0], B.shape[1]), order="F")
    _check(lib().or_matmul_optimized(_pd(A), _pd(B), A.shape[0], A.shape[1], B.shape[1],
                                     tile, workers, _pd(out)))
    return out


def symmetric_eig(G):
    G = _f64(G)
    m = G.shape[0]
    if G.shape[0] != G.shape[1]:
        raise OracleError(6, "symmetric_eig: matrix is not square")
    w = np.empty(m)
    V = np.empty((m, m), order="F")
    _check(lib().or_symmetric_eig(_pd(G), m, _pd(w), _pd(V)))
    return w, V


def jacobi_eig(G):
    G = _f64(G)
    m = G.shape[0]
    w = np.empty(m)
    V = np.empty((m, m), order="F")
    lib().or_jacobi_eig(_pd(G), m, _pd(w), _pd(V))
    return w, V


class Model:
    """Host TrainedModel (mset.hpp:46-57) as produced by the oracle."""

    def __init__(self, **kw):
        self.__dict__.update(kw)

    @property
    def memory_normalized(self):
        return self.D / self.scale[:, None]


def train(X, m, kind=INVERSE_DISTANCE, h=0.0, backend=REFERENCE, tile=64, workers=1):
    X = _f64(X)
    N, n = X.shape
    idx = np.empty(m, dtype=np.int64)
    D = np.empty((n, m), order="F")
    scale = np.empty(n)
    pinv = np.empty((m, m), order="F")
    spec = np.empty(m)
    rank = np.zeros(1, dtype=np.int64)
    hout = np.zeros(1)
    _check(lib().or_train(_pd(X), N, n, m, kind, h, backend, tile, workers, _pi64(idx),
                          _pd(D), _pd(scale), _pd(pinv), _pd(spec), _pi64(rank), _pd(hout)))
    return Model(source_indices=idx, D=D, scale=scale, gram_pinv=pinv,
                 eigen_spectrum=spec, rank=int(rank[0]), h=float(hout[0]), kind=kind)


def estimate(model, obs, backend=REFERENCE, tile=64, workers=1):
    obs = _f64(obs)
    N, n = obs.shape
    if n != model.D.shape[0]:
        raise OracleError(6, f"estimate: observation signal count {n} does not match "
                             f"model signal count {model.D.shape[0]}")
    est = np.empty((N, n), order="F")
    res = np.empty((N, n), order="F")
    D, sc, pv = _f64(model.D), _f64(model.scale), _f64(model.gram_pinv)
    _check(lib().or_estimate(_pd(D), _pd(sc), _pd(pv), n, D.shape[1], model.rank,
                             model.kind, model.h, _pd(obs), N, backend, tile, workers,
                             _pd(est), _pd(res)))
    return est, res


# --------------------------------------------------------------- sweep
def cell_data_seed(master, n, N, m, r):
    return lib().or_cell_data_seed(master, n, N, m, r)


def generate_cells(signal_counts, observation_counts, memory_counts):
    """sweep.cpp:103-117: signals-major, then memory, then observations."""
    cells = []
    for n in signal_counts:
        for m in memory_counts:
            for obs in observation_counts:
                cells.append(((n, obs, m), m >= 2 * n))
    return cells


# ------------------------------------------------------------ model files
def _json_double(v: float) -> str:
    """nlohmann::json number formatting: shortest round-trip, '.0' kept."""
    s = repr(float(v))
    return s


def save_model_csm1(model, path: str) -> None:
    """save_model (mset.cpp:229-267): "CSM1", u32 1, u64 n, u64 m,
    u32 kind (1 = gaussian), f64 bandwidth, u64 rank, D, gram_pinv,
    eigen_spectrum, signal_scale (column-major FP64), m x u64 source indices;
    plus the nlohmann dump(2) sidecar "<path>.json" (keys sorted)."""
    import struct
    D = _f64(model.D)
    n, m = D.shape
    with open(path, "wb") as f:
        f.write(b"CSM1")
        f.write(struct.pack("<IQQIdQ", 1, n, m, 1 if model.kind == GAUSSIAN else 0, model.h, model.rank))
        f.write(np.asarray(D, dtype="<f8").tobytes(order="F"))
        f.write(np.asarray(_f64(model.gram_pinv), dtype="<f8").tobytes(order="F"))
        f.write(np.asarray(model.eigen_spectrum, dtype="<f8").tobytes())
        f.write(np.asarray(model.scale, dtype="<f8").tobytes())
        f.write(np.asarray(model.source_indices, dtype="<u8").tobytes())
    kind = "gaussian" if model.kind == GAUSSIAN else "inverse_distance"
    with open(path + ".json", "w") as f:
        f.write("{\n  \"format\": \"CSM1\",\n  \"kernel\": {\n"
                f"    \"bandwidth\": {_json_double(model.h)},\n    \"kind\": \"{kind}\"\n  }},\n"
                f"  \"n_memory\": {m},\n  \"n_signals\": {n},\n  \"rank\": {model.rank},\n"
                "  \"version\": 1\n}\n")


def load_model_csm1(path: str):
    """load_model (mset.cpp:269-310); raises OracleError(8, ...) with the
    reference texts."""
    import struct
    try:
        data = open(path, "rb").read()
    except OSError:
        raise OracleError(8, f"load_model: cannot open {path}")
    if data[:4] != b"CSM1":
        raise OracleError(8, f"load_model: bad magic in {path}")
    if len(data) < 8 or struct.unpack_from("<I", data, 4)[0] != 1:
        raise OracleError(8, f"load_model: unsupported version in {path}")
    hdr = struct.calcsize("<IQQIdQ")
    if len(data) < 4 + hdr:
        raise OracleError(8, f"load_model: truncated file {path}")
    _, n, m, kind, h, rank = struct.unpack_from("<IQQIdQ", data, 4)
    off = 4 + hdr
    need = 8 * (n * m + m * m + m + n + m)
    if len(data) < off + need:
        raise OracleError(8, f"load_model: truncated file {path}")
    def take(count, dt="<f8"):
        nonlocal off
        a = np.frombuffer(data, dtype=dt, count=count, offset=off)
        off += 8 * count
        return a
    D = take(n * m).reshape((n, m), order="F").copy(order="F")
    pinv = take(m * m).reshape((m, m), order="F").copy(order="F")
    spec = take(m).copy()
    scale = take(n).copy()
    idx = take(m, "<u8").astype(np.int64)
    return Model(source_indices=idx, D=D, scale=scale, gram_pinv=pinv, eigen_spectrum=spec,
                 rank=int(rank), h=float(h), kind=GAUSSIAN if kind == 1 else INVERSE_DISTANCE)


# ------------------------------------------------------------------ SPRT
def sprt_params(sigma, k=3.0, alpha=1e-3, beta=1e-3):
    """Per-signal c = M / sigma^2, h = M / 2 with M = k sigma; Wald
    thresholds A = ln(beta / (1 - alpha)), B = ln((1 - beta) / alpha)."""
    import math
    sigma = np.asarray(sigma, dtype=np.float64)
    M = k * sigma
    c = M / (sigma * sigma)
    h = M / 2.0
    return c, h, math.log(beta / (1.0 - alpha)), math.log((1.0 - beta) / alpha)


def sprt(resid, c, h, A, B, state=None):
    """or_sprt: returns (flags N x n uint8 column-major, state (n, 2), counts (n, 2))."""
    r = _f64(resid)
    N, n = r.shape
    st = np.zeros((n, 2)) if state is None else np.array(state, dtype=np.float64).reshape(n, 2).copy()
    flags = np.zeros((N, n), dtype=np.uint8, order="F")
    counts = np.zeros((n, 2), dtype=np.int64)
    lib().or_sprt(_pd(r), N, n, max(N, 1), _pd(np.ascontiguousarray(c, dtype=np.float64)),
                  _pd(np.ascontiguousarray(h, dtype=np.float64)), A, B, _pd(st),
                  flags.ctypes.data_as(C.POINTER(C.c_uint8)), _pi64(counts))
    return flags, st, counts
