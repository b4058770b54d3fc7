"""CSM1 model files (save_model / load_model, mset.cpp:225-310).

CPU: the oracle's restated writer/reader round-trips bitwise and raises the
reference's IoError texts (port of test_mset.cpp:292-322 "model file
round-trip").  GPU: the library's writer is byte-identical to the oracle's
for the same model, a GPU-written file loads back into a model whose FP64
estimates are bitwise those of the original, and a file written from a CPU
(oracle) model drives the GPU FP64 path to the reference's bits.
"""
import json
import os

import numpy as np
import pytest


def _model(oracle):
    X = oracle.synthesize_uniform(3, 96, 0.3, 0.2, 1.0, 0.2, 3.5, 53)
    return oracle.train(X, 8, oracle.GAUSSIAN, 2.5)


def test_oracle_csm1_round_trip(oracle, tmp_path):
    m = _model(oracle)
    path = str(tmp_path / "model.csm")
    oracle.save_model_csm1(m, path)
    assert os.path.exists(path + ".json")
    side = json.load(open(path + ".json"))
    assert side == {"format": "CSM1", "kernel": {"bandwidth": 2.5, "kind": "gaussian"},
                    "n_memory": 8, "n_signals": 3, "rank": m.rank, "version": 1}
    lo = oracle.load_model_csm1(path)
    assert lo.rank == m.rank and lo.kind == m.kind and lo.h == m.h
    assert lo.source_indices.tolist() == m.source_indices.tolist()
    assert lo.D.tobytes(order="F") == np.asfortranarray(m.D).tobytes(order="F")
    assert lo.gram_pinv.tobytes(order="F") == np.asfortranarray(m.gram_pinv).tobytes(order="F")
    obs = oracle.synthesize_uniform(3, 20, 0.3, 0.2, 1.0, 0.2, 3.5, 59)
    a = oracle.estimate(m, obs)[0]
    b = oracle.estimate(lo, obs)[0]
    assert np.array_equal(a, b)
    # header: 4 magic + u32 + 2 u64 + u32 + f64 + u64, then the arrays
    assert os.path.getsize(path) == 44 + 8 * (3 * 8 + 64 + 8 + 3 + 8)


def test_oracle_csm1_errors(oracle, tmp_path):
    path = str(tmp_path / "bad.csm")
    open(path, "wb").write(b"XXXX")
    with pytest.raises(oracle.OracleError, match="load_model: bad magic in"):
        oracle.load_model_csm1(path)
    open(path, "wb").write(b"CSM1" + (2).to_bytes(4, "little"))
    with pytest.raises(oracle.OracleError, match="load_model: unsupported version in"):
        oracle.load_model_csm1(path)
    oracle.save_model_csm1(_model(oracle), path)
    data = open(path, "rb").read()
    open(path, "wb").write(data[:-5])
    with pytest.raises(oracle.OracleError, match="load_model: truncated file"):
        oracle.load_model_csm1(path)
    with pytest.raises(oracle.OracleError, match="load_model: cannot open"):
        oracle.load_model_csm1(str(tmp_path / "missing.csm"))


@pytest.mark.gpu
def test_gpu_csm1_byte_identical_and_round_trip(oracle, tmp_path):
    import paper_2003_08011_b200 as p
    B = p.BackendId("b200", 0, "fp64")
    X = oracle.synthesize_uniform(3, 96, 0.3, 0.2, 1.0, 0.2, 3.5, 53)
    obs = oracle.synthesize_uniform(3, 20, 0.3, 0.2, 1.0, 0.2, 3.5, 59)
    g = p.train(X, 8, p.KernelConfig(p.KernelKind.gaussian, 2.5), B)
    path = str(tmp_path / "gpu.csm")
    p.save_model(g, path)
    e = g.export()
    ref = oracle.Model(source_indices=e["source_indices"], D=e["D"], scale=e["signal_scale"],
                       gram_pinv=e["gram_pinv"], eigen_spectrum=e["eigen_spectrum"], rank=g.rank,
                       h=g.kernel.bandwidth, kind=oracle.GAUSSIAN)
    opath = str(tmp_path / "oracle.csm")
    oracle.save_model_csm1(ref, opath)
    assert open(path, "rb").read() == open(opath, "rb").read()
    assert open(path + ".json").read() == open(opath + ".json").read()
    loaded = p.load_model(path, B)
    assert loaded.rank == g.rank
    assert np.array_equal(p.estimate(loaded, obs).estimates, p.estimate(g, obs).estimates)
    # CPU-trained model file -> GPU FP64 estimate: the reference's bits
    cpu = oracle.train(X, 8, oracle.GAUSSIAN, 2.5)
    cpath = str(tmp_path / "cpu.csm")
    oracle.save_model_csm1(cpu, cpath)
    want = oracle.estimate(cpu, obs)[0]
    got = p.estimate(p.load_model(cpath, B), obs).estimates
    assert np.abs(got - want).max() <= 1e-14 * np.abs(want).max()  # Gaussian: CUDA exp vs glibc
    cpu_i = oracle.train(X, 8)
    oracle.save_model_csm1(cpu_i, cpath)
    assert np.array_equal(p.estimate(p.load_model(cpath, B), obs).estimates, oracle.estimate(cpu_i, obs)[0])
    # errors carry the reference texts
    open(cpath, "wb").write(b"NOPE")
    with pytest.raises(p.IoError, match="load_model: bad magic in"):
        p.load_model(cpath, B)
    with pytest.raises(p.IoError, match="load_model: cannot open"):
        p.load_model(str(tmp_path / "missing.csm"), B)
