"""C++-level drop-in: the unmodified reference's nbb::Simulation and the GPU
engine behind include/nbbgpu.hpp, in one process, byte-identical after every step
(oracle/cpp_dropin_check.cpp, built by oracle/Makefile where /root/reference exists
and shipped prebuilt in oracle/_ref)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "dropin_check")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(EXE), reason="oracle/_ref/dropin_check not built")
def test_cpp_dropin_lockstep():
    out = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.startswith("OK"), out.stdout
