"""Multi-rank path on CPU: world_size 2 and 3 over gloo (127.0.0.1).

Each rank runs the C oracle on its owned partition rows only
(step_compact_linear over [lo, hi), the reference's chunked parallel_for,
stencil.cpp:236-260) and exchanges exactly the halo bytes the host planner
(nbbgpu_plan_partition / nbbgpu_plan_needs, the same code the GPU path uses)
lists, through paper_2110_12952_b200.distributed.exchange.  The summed partial
state hashes and the owned bytes must equal the single-process run after every
step -- acceptance C9's determinism across worker counts, across ranks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


CASES = [
    # (name, k, s, replicas, level, rule(birth, survive, moore), steps)
    ("sierpinski-triangle", 3, 2, [(0, 0), (1, 0), (0, 1)], 9, (8, 12, True), 6),
    ("sierpinski-triangle", 3, 2, [(0, 0), (1, 0), (0, 1)], 5, (0x48, 0x1C, False), 5),
    ("sierpinski-carpet", 8, 3, [(0, 0), (1, 0), (2, 0), (0, 1), (2, 1), (0, 2), (1, 2), (2, 2)], 4,
     (8, 12, True), 4),
    ("vicsek", 5, 3, [(1, 0), (0, 1), (1, 1), (2, 1), (1, 2)], 5, (0x6, 0x9, True), 4),
]


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2110_12952_b200.descriptor import FractalDescriptor
    from paper_2110_12952_b200.distributed import PartitionPlan, exchange, wrap_u64_sum
    try:
        for name, k, s, rep, level, (birth, survive, moore), steps in CASES:
            d = FractalDescriptor(name, k, s, rep)
            plan = PartitionPlan(d, level, rank, world)
            o = oracle.Oracle(rep, k, s, level)
            o.seed(77, 0.45)
            ref = oracle.Oracle(rep, k, s, level)
            ref.seed(77, 0.45)
            for step in range(steps):
                o.step_range(birth, survive, moore, plan.lo, plan.hi)
                o.swap()

                def pack(p):
                    return torch.from_numpy(o.front[plan.send[p].astype(np.int64)].copy())

                def unpack(p, buf):
                    o.front[plan.recv[p].astype(np.int64)] = buf.numpy()

                exchange(plan, dist, pack, lambda p, n: torch.empty(n, dtype=torch.uint8), unpack)
                ref.step(birth, survive, moore)
                part = o.state_hash_range(plan.lo, plan.hi)
                t = torch.tensor([part & 0xFFFFFFFF, part >> 32], dtype=torch.int64)
                parts = [torch.zeros_like(t) for _ in range(world)]
                dist.all_gather(parts, t)
                total = wrap_u64_sum(int(x[0]) | (int(x[1]) << 32) for x in parts)
                assert total == ref.state_hash(), (name, level, step)
                assert np.array_equal(o.front[plan.lo:plan.hi], ref.front[plan.lo:plan.hi]), (name, step)
        q.put((rank, "ok"))
    except Exception as e:  # report to the parent
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_halo_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, msg in results:
        assert msg == "ok", f"rank {rank}:\n{msg}"


def test_plan_lists_are_symmetric_and_disjoint():
    import sys
    sys.path.insert(0, ROOT)
    from paper_2110_12952_b200.descriptor import builtin_descriptor
    from paper_2110_12952_b200.distributed import PartitionPlan
    T = builtin_descriptor("sierpinski-triangle")
    n = 4
    plans = [PartitionPlan(T, 12, r, n) for r in range(n)]
    for r, pl in enumerate(plans):
        for p in pl.peers:
            assert np.array_equal(pl.send[p], plans[p].recv[r])
            # everything I send is mine, everything I receive is not
            assert ((pl.send[p] >= pl.lo) & (pl.send[p] < pl.hi)).all()
            assert not ((pl.recv[p] >= pl.lo) & (pl.recv[p] < pl.hi)).any()
    # the triangle's halo is tiny: sub-triangles touch at corners only
    assert max(pl.halo_bytes() for pl in plans) < 0.02 * (3 ** 12) / n
