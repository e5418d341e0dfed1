"""The C-ABI library loads and exports every symbol include/zsvd.h declares
(no compute calls here), and the host mirror fails loudly without a device."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "zsvd.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(zsvd_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_header():
    from paper_1805_00754_b200 import _capi
    L = _capi.lib()
    syms = header_symbols()
    assert len(syms) >= 40
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    # the Python binding declares exactly the header's functions
    assert sorted(_capi.SIGNATURES) == syms
    assert b"sm_100a" in L.zsvd_version()


def test_library_is_sm100a_cubin():
    so = os.path.join(ROOT, "paper_1805_00754_b200", "libzsvd.so")
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_oracle_not_used_by_product():
    """The product package never imports, loads or links the oracle."""
    pkg = os.path.join(ROOT, "paper_1805_00754_b200")
    bad = re.compile(r"^\s*(import\s+oracle|from\s+oracle|.*liboracle|.*zsvd_oracle\.h|.*CDLL\(.*oracle)", re.M)
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cpp", ".cuh")):
                src = open(os.path.join(dirpath, f)).read()
                assert not bad.search(src), f


def test_no_device_fails_loudly():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("device present")
    import paper_1805_00754_b200 as z
    with pytest.raises(z.CudaError):
        z.BlockStore(4, 3, 1.0)
    with pytest.raises(z.CudaError):
        z.thin_svd([[1.0, 2.0], [3.0, 4.0]])


def test_parameter_errors_precede_device():
    import paper_1805_00754_b200 as z
    with pytest.raises(z.InvalidParameterError):
        z.BlockStore(0, 5, 0.98)
    with pytest.raises(z.InvalidParameterError):
        z.BlockStore(5, 0, 0.98)
    with pytest.raises(z.InvalidParameterError):
        z.BlockStore(5, 5, 0.0)
    with pytest.raises(z.InvalidParameterError):
        z.BlockStore(5, 5, 1.5)
