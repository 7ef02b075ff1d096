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


@pytest.mark.gpu
def test_cpp_shim_amr_at_the_papers_sizes(gpu_lib):
    """run_amr on the reference's built-in cases with their own step schedules
    at the paper's AMR configuration (base 64^2 / 8^3): lax_liu_6 at 512^2 and
    1024^2 (640 and 1280 steps), ellipsoid3d at 64^3 and 128^3; the reference
    runs beside the device run on the box's host (about 1.5 minutes)."""
    if not os.path.exists(BIN):
        pytest.skip("shim_parity not built (needs /root/reference at build time)")
    r = subprocess.run([BIN, "amr-full"], capture_output=True, text=True, timeout=1500)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "SHIM PARITY OK" in r.stdout
