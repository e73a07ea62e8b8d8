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


# ---- the reference itself with the GPU backends compiled in (gpu_backend.patch) ----
GPU_DIR = os.path.join(ROOT, "oracle", "_ref", "gpu")


def _run(args, env=None, timeout=900):
    exe = os.path.join(GPU_DIR, args[0])
    assert os.path.exists(exe), f"{exe} missing: build with `make -C oracle` where /root/reference exists"
    e = dict(os.environ)
    e.update(env or {})
    out = subprocess.run([exe] + args[1:], capture_output=True, text=True, timeout=timeout, env=e)
    return out.returncode, out.stdout + out.stderr


@pytest.mark.parametrize("part", ["names", "run_simulation", "lockstep", "errors", "verify_stencil", "bench_run",
                                  "determinism"])
def test_reference_callers_on_gpu_backends(part):
    # parse_backend, run_simulation, Simulation + front(), errors, verify_stencil with a
    # LockstepHook fault, bench_run (incl. acceptance C8 under the 2 GiB cap), the C9
    # generator -- all through the reference's unchanged entry points
    rc, log = _run(["gpu_callers", part])
    assert rc == 0 and "OK: 0 failure(s)" in log, log[-4000:]
    assert "[FAIL]" not in log


def test_reference_acceptance_unchanged_with_adapter():
    # the patched library keeps every CPU behaviour: acceptance C1-C9 unchanged
    rc, log = _run(["acceptance"])
    assert rc == 0 and log.count("[PASS]") == 9, log[-4000:]


@pytest.mark.parametrize("substitute", ["compact", "bb", "compact,bb"])
def test_reference_acceptance_on_gpu(substitute):
    # the UNMODIFIED acceptance.cpp with its Backend::Compact (and/or BoundingBox)
    # simulations running on the GPU engine: C5 (verify_stencil lockstep + 50
    # randomized trials), C8 (memory-cap bench_run) and C9 (run_simulation
    # determinism) drive the GPU
    rc, log = _run(["acceptance"], env={"NBB_GPU_SUBSTITUTE": substitute})
    assert rc == 0 and log.count("[PASS]") == 9, log[-4000:]
