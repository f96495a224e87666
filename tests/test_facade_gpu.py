"""GPU: the C++ drop-in facade (include/rnnwave/engine.hpp) used the way the reference's own
tests use rnnwave::Engine (tests/cpp/facade_parity.cpp), checked against the C restatement
of the reference with the SURVEY §8c tolerances."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def test_cpp_facade_parity():
    exe = os.path.join(HERE, "cpp", "build", "facade_parity")
    if not os.path.exists(exe):
        subprocess.run(["sh", os.path.join(HERE, "cpp", "build.sh")], check=True, capture_output=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(out.stdout[-6000:])
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    assert "FACADE PASS" in out.stdout
