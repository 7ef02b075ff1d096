"""Drop-in check: the reference's own entry points (run_uniform, step_block,
run_mr on its built-in cases) vs the same calls through the C++ shim
paper_1603_05211_b200/host/adaptflow_gpu.hpp -> libafgpu.so. The binary is
built in the build container (it needs the reference headers) by
`make -C oracle shim` and travels to the GPU box."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "shim_parity")


@pytest.mark.gpu
def test_cpp_shim_bit_identical_to_reference(gpu_lib):
    if not os.path.exists(BIN):
        pytest.skip("shim_parity not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "SHIM PARITY OK" in r.stdout
