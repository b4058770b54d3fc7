"""CPU-side checks of the product library (no GPU needed).

* the C-ABI library builds/loads and exports every symbol include/cstress_b200.h
  declares;
* the host data feed (synthesize, seed derivation) matches the oracle
  bit-for-bit;
* backend-id parsing / labels and host-side validation behave like the
  reference (backends.cpp:77-111).
"""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "cstress_b200.h")).read()
    decl = r"^\s*(?:cs_status|const char\*|uint64_t)\s+(cs_[a-z0-9_]+)\s*\("
    return sorted(set(re.findall(decl, text, flags=re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2003_08011_b200 import _lib
    L = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    # the python binding covers the whole header
    assert set(syms) <= set(_lib.exported_symbols())


def test_library_is_sm100a():
    import subprocess
    from paper_2003_08011_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_synthesize_matches_oracle_bitwise(oracle):
    import paper_2003_08011_b200 as p
    for args in [(1, 500, 0.0, 0.0, 1.0, 0.0, 3.0, 7), (5, 3000, 0.5, 0.3, 1.0, 0.5, 4.0, 123),
                 (20, 400, 0.3, 0.2, 1.0, 0.2, 3.5, 99), (3, 64, 0.8, 0.9, 2.0, 1.0, 5.0, 1)]:
        a = p.synthesize(p.SignalSpec.uniform(*args)).data
        b = oracle.synthesize_uniform(*args)
        assert a.tobytes() == b.tobytes()


def test_synthesize_errors_match_reference_classes():
    import paper_2003_08011_b200 as p
    with pytest.raises(p.MomentInfeasible, match="Fleishman"):
        p.synthesize(p.SignalSpec.uniform(2, 32, 0.0, 0.0, 1.0, 2.0, 6.0, 1))
    with pytest.raises(p.MomentInfeasible, match="Pearson bound"):
        p.synthesize(p.SignalSpec.uniform(2, 32, 0.0, 0.0, 1.0, 0.0, 1.0, 1))
    with pytest.raises(p.ConfigError):
        p.synthesize(p.SignalSpec.uniform(2, 32, 1.0, 0.0, 1.0, 0.0, 3.0, 1))


def test_seed_derivation_matches_oracle(oracle):
    import paper_2003_08011_b200 as p
    assert p.cell_data_seed(20260810, 100, 100000, 1000, 3) == oracle.cell_data_seed(
        20260810, 100, 100000, 1000, 3)
    assert p.derive_seed(5, [0]) == oracle.derive_seed(5, [0])


def test_backend_ids_parse_and_validate():
    import paper_2003_08011_b200 as p
    b = p.BackendId("b200", 3, "fp32")
    assert b.label() == "b200[device=3/precision=fp32]"
    assert p.BackendId.parse(b.label()) == b
    assert p.BackendId.parse("b200") == p.BackendId()
    with pytest.raises(p.ConfigError):
        p.BackendId.parse("gpu")
    with pytest.raises(p.ConfigError):
        p.BackendId("b200", 0, "fp16").validate()
    with pytest.raises(p.ConfigError):
        p.KernelConfig(p.KernelKind.gaussian, -1.0).validate()


def test_algorithm_registry():
    import paper_2003_08011_b200 as p
    assert p.algorithm_by_name("mset2").name() == "mset2"
    assert p.algorithm_by_name("mean").name() == "mean"
    with pytest.raises(p.ConfigError):
        p.algorithm_by_name("svm")


def test_cpp_host_layer_compiles_and_links():
    """include/cstress_b200.hpp (C++ mirror of the reference API) builds
    against the library; the test program lists its cases without a GPU."""
    import subprocess
    from paper_2003_08011_b200 import build as b
    exe = b.build_cpp_test()
    out = subprocess.run([exe, "--list"], capture_output=True, text=True, check=True).stdout
    assert "train / estimate" in out and "plugin contract" in out
