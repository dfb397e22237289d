"""CPU-side checks of the C-ABI library: it builds for sm_100a, loads, and exports
every entry point include/ibgm.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "ibgm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ib_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = _declared()
    for need in ("ib_create", "ib_set_boundary", "ib_step", "ib_get_fields", "ib_destroy"):
        assert need in names


def test_library_builds_loads_and_exports_every_symbol():
    from paper_1305_3976_b200 import _build, ibgm
    path = _build.build()
    L = ctypes.CDLL(path)
    for name in _declared():
        assert hasattr(L, name), name
    assert set(_declared()) == set(ibgm.SYMBOLS)


def test_library_is_sm100a_code():
    from paper_1305_3976_b200 import _build
    path = _build.build()
    out = subprocess.run(["cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_oracle_is_not_on_the_product_path():
    """The product package never imports or links the oracle."""
    pkg = os.path.join(ROOT, "paper_1305_3976_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).lower() or f == "inputs.py", f


def test_invalid_arguments_fail_loudly_without_gpu():
    """Argument validation happens before any CUDA call."""
    from paper_1305_3976_b200 import ibgm
    with pytest.raises(ibgm.IBGMError) as e:
        ibgm.Context(4, 32, 0.01, 1.0, 1e-3)
    assert e.value.code == -1
    with pytest.raises(ibgm.IBGMError):
        ibgm.Context(2, 17, 0.01, 1.0, 1e-3)   # no admissible line segmentation
    with pytest.raises(ibgm.IBGMError):
        ibgm.Context(2, 32, 0.01, 1.0, -1.0)
