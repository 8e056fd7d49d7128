"""The C++ drop-in (include/sphere_gpu.hpp over libsphgpu.so) executed on the B200
against the reference's own fp64 outputs and known answers (tests/cpp/shim_pins.cpp,
built with the unmodified reference headers by tests/cpp/build.sh)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_bin", "shim_pins")


def test_cpp_dropin_pins_run_on_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    if not os.path.exists(BIN):
        if os.path.isdir("/root/reference/proj/include"):
            subprocess.run([os.path.join(ROOT, "tests", "cpp", "build.sh")], check=True)
        else:
            pytest.fail("tests/cpp/_bin/shim_pins was not built (run __graft_entry__.build() where the "
                        "reference headers are)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "0 failed" in r.stdout, r.stdout
