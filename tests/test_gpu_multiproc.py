"""The multi-rank bench path on ONE GPU: torchrun with 2 and 3 processes sharing
cuda:0 (gloo between them, halo words staged through the host), packed kernel,
partitioned groups and the per-step boundary-word exchange of
DistributedSimulation.  The final state hash must equal the single-process run of
the same steps (acceptance C9 across rank counts)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(nproc, level, port):
    args = ["bench.py", "--level", str(level), "--steps", "4", "--warmup", "3", "--no-e2e",
            "--no-cpu-baseline"]
    if nproc > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
               "--master-addr", "127.0.0.1", "--master-port", str(port)] + args + [
               "--gpus", str(nproc), "--dist-backend", "gloo", "--transport", "torch", "--device", "0"]
    else:
        cmd = [sys.executable] + args
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    line = [l for l in out.stdout.splitlines() if l.startswith("{")][-1]
    return json.loads(line)


@pytest.mark.parametrize("nproc", [2, 3])
def test_multirank_bench_matches_single(nproc):
    single = _bench(1, 14, 0)
    multi = _bench(nproc, 14, 29517 + nproc)
    assert multi["final_state_hash"] == single["final_state_hash"]
    assert multi["n_gpus"] == nproc and "packed" in multi["config"]["kernel"]
