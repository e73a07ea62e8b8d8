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


def _bench(nproc, level, port, transport="torch"):
    args = ["bench.py", "--level", str(level), "--steps", "4", "--warmup", "3", "--no-e2e",
            "--no-cpu-baseline"]
    if nproc > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
               "--master-addr", "127.0.0.1", "--master-port", str(port)] + args + [
               "--gpus", str(nproc), "--dist-backend", "gloo", "--transport", transport, "--device", "0"]
    else:
        cmd = [sys.executable] + args
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    line = [l for l in out.stdout.splitlines() if l.startswith("{")][-1]
    return json.loads(line)


@pytest.mark.parametrize("nproc", [2, 3])
def test_multirank_bench_matches_single(nproc):  # torch.distributed point-to-point (gloo)
    single = _bench(1, 14, 0)
    multi = _bench(nproc, 14, 29517 + nproc)
    assert multi["final_state_hash"] == single["final_state_hash"]
    # ranks sharing cuda:0: one GPU stepped, nproc partitions
    assert multi["n_gpus"] == 1 and multi["engine"]["partitions"] == nproc
    assert "packed" in multi["engine"]["kernel"]


@pytest.mark.parametrize("nproc", [2, 3])
def test_multirank_p2p_transport_matches_single(nproc):
    # the peer-memory transport (CUDA IPC mappings of the boundary planes, pushes +
    # system-scope arrival counters): several processes on ONE GPU exercise the
    # same IPC / counter protocol the NVLink peers use
    single = _bench(1, 14, 0)
    multi = _bench(nproc, 14, 29617 + nproc, transport="p2p")
    assert multi["final_state_hash"] == single["final_state_hash"]
    multi20 = _bench(nproc, 16, 29717 + nproc, transport="p2p")
    assert multi20["final_state_hash"] == _bench(1, 16, 0)["final_state_hash"]


def test_multirank_auto_transport_picks_p2p():
    out = _bench(2, 12, 29817, transport="auto")
    assert "halo transport p2p" in out["engine"]["parallelism"]
    assert out["final_state_hash"] == _bench(1, 12, 0)["final_state_hash"]


def test_bench_gpus_without_torchrun_relaunches():
    # `bench.py --gpus 2` (no torchrun): re-launched as 2 ranks; pinned to one device
    # here, so the line reports 2 partitions on 1 GPU -- never n_gpus 2
    cmd = [sys.executable, "bench.py", "--level", "14", "--steps", "4", "--warmup", "3", "--no-e2e",
           "--no-cpu-baseline", "--gpus", "2", "--dist-backend", "gloo", "--transport", "p2p", "--device", "0"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 1 and line["engine"]["partitions"] == 2
    assert line["final_state_hash"] == _bench(1, 14, 0)["final_state_hash"]


def test_bench_gpus_refuses_without_devices():
    import torch
    n = torch.cuda.device_count() + 1
    out = subprocess.run([sys.executable, "bench.py", "--gpus", str(n), "--steps", "3"], cwd=ROOT,
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 2
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert "error" in line and line["n_gpus"] == n - 1


def test_multirank_p2p_in_kernel_halo_r18():
    # r=18 picks q=8 with <= 4096 groups per rank: the step kernel gathers the halo
    # words itself after waiting on the peers' arrival counter
    single = _bench(1, 18, 0)
    multi = _bench(2, 18, 29917, transport="p2p")
    assert multi["final_state_hash"] == single["final_state_hash"]
