"""Host-side planning of the packed layout (no GPU): every admissible packed tile
level of the built-in and descriptor-file fractals builds its plan (halo slots,
boundary sources, micro-block external tables), and the partition lists cover
exactly the cross-rank halo links."""
import numpy as np
import pytest

from paper_2110_12952_b200 import builtin_descriptor
from paper_2110_12952_b200.descriptor import FractalDescriptor
from paper_2110_12952_b200.distributed import (PartitionPlan, packed_elem_cells, packed_info,
                                               plan_packed_level)

T = builtin_descriptor("sierpinski-triangle")
CARPET = builtin_descriptor("sierpinski-carpet")
VICSEK = builtin_descriptor("vicsek")
H = FractalDescriptor("h", 7, 3, [(0, 0), (2, 0), (0, 1), (1, 1), (2, 1), (0, 2), (2, 2)])
Y = FractalDescriptor("y", 12, 4, [(1, 0), (2, 0), (0, 1), (1, 1), (2, 1), (3, 1), (0, 2),
                                  (1, 2), (2, 2), (3, 2), (1, 3), (2, 3)])


@pytest.mark.parametrize("desc,r,qs", [(T, 9, (2, 4, 6, 8)), (T, 20, (8,)), (CARPET, 5, (2, 4)),
                                       (VICSEK, 5, (2, 4)), (H, 5, (2, 4)), (Y, 5, (2, 4))])
def test_plans_build(desc, r, qs):
    for q in qs:
        info = packed_info(desc, r, q)
        assert info["q"] == q and info["C"] == desc.k ** q
        assert info["NG"] == (info["T"] + 31) // 32
        assert info["T"] * info["C"] == desc.k ** r


def test_default_levels():
    assert plan_packed_level(T, 20) == 8
    assert plan_packed_level(T, 16) == 8
    assert plan_packed_level(CARPET, 9) == 4
    assert plan_packed_level(T, 1) == -1


def _neighbours(desc, r):
    """compact offset -> list of compact offsets of its fractal neighbours (Moore)."""
    import oracle
    o = oracle.Oracle(desc.replicas, desc.k, desc.s, r)
    w = desc.k ** ((r + 1) // 2)
    n = desc.k ** r
    nb = []
    for i in range(n):
        x, y = o.to_embedded(i % w, i // w)
        lst = []
        for dx, dy in [(1, 0), (-1, 0), (0, 1), (0, -1), (1, 1), (1, -1), (-1, 1), (-1, -1)]:
            if not (0 <= x + dx < o.side and 0 <= y + dy < o.side):
                continue
            c = o.to_compact(x + dx, y + dy)
            if c is not None:
                lst.append(c[1] * w + c[0])
        nb.append(lst)
    return nb


@pytest.mark.parametrize("desc,r,q,nranks", [(T, 7, 2, 3), (T, 8, 4, 2), (CARPET, 4, 2, 3),
                                             (VICSEK, 5, 2, 2), (H, 4, 2, 3)])
def test_packed_partition_covers_halo(desc, r, q, nranks):
    nb = _neighbours(desc, r)
    plans = [PartitionPlan(desc, r, k, nranks, tile_level=q, packed=True) for k in range(nranks)]
    masks = [p.owned_cell_mask() for p in plans]
    assert np.array_equal(sum(m.astype(int) for m in masks), np.ones(desc.k ** r, dtype=int))
    for rank, plan in enumerate(plans):
        got = set()
        for peer, elems in plan.recv.items():
            cells = packed_elem_cells(desc, r, q, elems)
            assert all(masks[peer][c] for c in cells)  # only the peer's cells
            got.update(int(c) for c in cells)
            # symmetric: what I receive from peer is what peer sends me
            assert np.array_equal(np.sort(plans[peer].send[rank]), np.sort(elems))
        need = {j for i in np.nonzero(masks[rank])[0] for j in nb[i] if not masks[rank][j]}
        assert need <= got, f"rank {rank}: {len(need - got)} foreign neighbours not covered"
