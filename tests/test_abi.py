"""CPU tests of the drop-in boundary: libafgpu.so builds for sm_100a, loads,
exports exactly the functions include/af_gpu.h declares, and its host-only
entry points agree with the oracle. No kernel is launched here."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "af_gpu.h")


def declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(af_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_1603_05211_b200 import _abi
    lib = _abi.load()
    names = declared_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    # and the Python binding covers the whole header
    assert set(names) <= set(_abi.SIGNATURES), set(names) - set(_abi.SIGNATURES)
    out = subprocess.run(["nm", "-D", "--defined-only", _abi.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (af_[a-z0-9_]+)$", out, flags=re.M))
    assert set(names) <= exported


def test_library_is_sm100a():
    from paper_1603_05211_b200 import _abi
    out = subprocess.run(["cuobjdump", "--list-elf", _abi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_case_fill_matches_oracle(oracle):
    from paper_1603_05211_b200 import uniform as U
    for kind, level in ((0, 6), (1, 5), (2, 4), (3, 4)):
        assert np.array_equal(U.case_fill(kind, 77, level), oracle.case_fill(kind, 77, level))


def test_errors_map_to_reference_exceptions():
    from paper_1603_05211_b200 import errors as E
    with pytest.raises(E.NonPhysicalState):
        E.raise_status(1, "x")
    with pytest.raises(E.RegisterMismatch):
        E.raise_status(2, "x")
    with pytest.raises(E.ConfigError):
        E.raise_status(8, "x")
    E.raise_status(0, "")


def test_no_cpu_fallback_without_gpu():
    """Without a visible GPU the solver must fail loudly, not compute on CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1603_05211_b200 import uniform as U
    from paper_1603_05211_b200.errors import DeviceError
    with pytest.raises(DeviceError):
        U.UniformSolver(2, 6)


def test_state_buffers_are_validated_before_the_abi():
    """Host states reach the C ABI as raw pointers to cells x 5 doubles, so the
    Python mirror rejects any other shape, dtype or layout first."""
    import numpy as np
    import pytest as _pt
    from paper_1603_05211_b200.uniform import _state_ptr
    cells = 64
    ok = np.zeros((cells, 5))
    assert _state_ptr(ok, cells) == ok.ctypes.data
    assert _state_ptr(np.zeros(cells * 5), cells)
    for bad in (np.zeros((cells, 4)), np.zeros((cells - 1, 5)), np.zeros((cells, 5), np.float32),
                np.zeros((5, cells)).T, np.zeros(cells * 5 - 1)):
        with _pt.raises((ValueError, TypeError)):
            _state_ptr(bad, cells)
