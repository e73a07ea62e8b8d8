"""Multi-GPU partitioning with a per-step halo exchange (north-star item 4).

One process per GPU.  Every rank keeps a full-size compact state, updates only
its contiguous range of partition rows (tile rows of k^(q/2) compact rows, or
compact rows when no tile level applies) and, after each step, exchanges the
halo bytes: the source cells of the tile-halo links that cross a partition
boundary (partition.inc).  The lists are computed on the host once and need no
communication: what rank p needs from me is exactly plan_needs(rank=p, peer=me).

The transport is torch.distributed point-to-point (NCCL over NVLink on the GPU
box, gloo in the CPU tests) with grouped isend/irecv, so the same host logic is
exercised by both.  The partial state hashes add up to the global hash
(Simulation::state_hash is an order-independent wrapping sum, stencil.cpp:196-234).
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field
from typing import Callable, Dict, List

import numpy as np

from . import _abi
from .descriptor import FractalDescriptor
from .errors import OutOfDomain
from .stencil import Neighborhood, StencilRule


def _needs(desc: FractalDescriptor, level: int, tile_level: int, rank: int, nranks: int,
           peer: int) -> np.ndarray:
    L = _abi.lib()
    rep = _abi.replica_array(desc.replicas)
    cnt = C.c_uint64()
    _abi.check(L.nbbgpu_plan_needs(rep, desc.k, desc.s, level, tile_level, rank, nranks, peer,
                                   None, C.byref(cnt)))
    out = np.zeros(max(1, cnt.value), dtype=np.uint64)
    _abi.check(L.nbbgpu_plan_needs(rep, desc.k, desc.s, level, tile_level, rank, nranks, peer,
                                   out.ctypes.data, C.byref(cnt)))
    return out[:cnt.value]


def _packed_needs(desc: FractalDescriptor, level: int, tile_level: int, rank: int, nranks: int,
                  peer: int) -> np.ndarray:
    L = _abi.lib()
    rep = _abi.replica_array(desc.replicas)
    cnt = C.c_uint64()
    _abi.check(L.nbbgpu_plan_packed_needs(rep, desc.k, desc.s, level, tile_level, rank, nranks, peer,
                                          None, C.byref(cnt)))
    out = np.zeros(max(1, cnt.value), dtype=np.uint64)
    _abi.check(L.nbbgpu_plan_packed_needs(rep, desc.k, desc.s, level, tile_level, rank, nranks, peer,
                                          out.ctypes.data, C.byref(cnt)))
    return out[:cnt.value]


def plan_packed_level(desc: FractalDescriptor, level: int) -> int:
    q = C.c_int()
    _abi.check(_abi.lib().nbbgpu_plan_packed_level(_abi.replica_array(desc.replicas), desc.k, desc.s,
                                                   level, C.byref(q)))
    return q.value


def packed_info(desc: FractalDescriptor, level: int, tile_level: int = -1) -> dict:
    """Packed plan geometry (nbbgpu_plan_packed)."""
    info = (C.c_int64 * 12)()
    _abi.check(_abi.lib().nbbgpu_plan_packed(_abi.replica_array(desc.replicas), desc.k, desc.s, level,
                                             tile_level, info))
    keys = ["q", "wq", "C", "Cp", "nH", "nSrc", "T", "NG", "Wc", "Hc", "nD", "wide"]
    return dict(zip(keys, [int(v) for v in info]))


def packed_elem_cells(desc: FractalDescriptor, level: int, tile_level: int, elems: np.ndarray) -> np.ndarray:
    """Compact byte offsets of the cells held by boundary-plane elements."""
    elems = np.ascontiguousarray(elems, dtype=np.uint64)
    out = np.zeros(max(1, 32 * elems.size), dtype=np.uint64)
    cnt = C.c_uint64()
    _abi.check(_abi.lib().nbbgpu_plan_packed_elem_cells(
        _abi.replica_array(desc.replicas), desc.k, desc.s, level, tile_level,
        elems.ctypes.data if elems.size else None, elems.size, out.ctypes.data, C.byref(cnt)))
    return out[:cnt.value]


def plan_tile_level(desc: FractalDescriptor, level: int) -> int:
    q = C.c_int()
    _abi.check(_abi.lib().nbbgpu_plan_tile_level(_abi.replica_array(desc.replicas), desc.k, desc.s,
                                                 level, C.byref(q)))
    return q.value


@dataclass
class PartitionPlan:
    """Owned range and halo lists of one rank (host only, no GPU).

    Byte layouts: lo/hi = owned compact byte range, halo elements = state bytes at
    compact byte offsets.  packed=True (the PACKED kernel): lo/hi = owned group
    range [g0, g1), halo elements = 32-bit boundary-plane words (g * nSrc + m)."""
    desc: FractalDescriptor
    level: int
    rank: int
    nranks: int
    tile_level: int = -1
    packed: bool = False
    lo: int = 0
    hi: int = 0
    recv: Dict[int, np.ndarray] = field(default_factory=dict)  # elements I need from peer
    send: Dict[int, np.ndarray] = field(default_factory=dict)  # elements peer needs from me

    @property
    def elem_bytes(self) -> int:
        return 4 if self.packed else 1

    def owned_cell_mask(self) -> np.ndarray:
        """Boolean mask over the compact byte layout of the cells this rank owns."""
        L = _abi.lib()
        rep = _abi.replica_array(self.desc.replicas)
        w = self.desc.k ** ((self.level + 1) // 2)
        h = self.desc.k ** (self.level // 2)
        mask = np.zeros(w * h, dtype=bool)
        if not self.packed:
            mask[self.lo:self.hi] = True
            return mask
        info = packed_info(self.desc, self.level, self.tile_level)
        wq, Wc, Hc, T = info["wq"], info["Wc"], info["Hc"], info["T"]
        tiles = np.zeros(Wc * Hc, dtype=bool)
        tiles[self.lo * 32:min(self.hi * 32, T)] = True
        m = np.repeat(np.repeat(tiles.reshape(Hc, Wc), wq, axis=0), wq, axis=1)
        return m.reshape(-1)

    def __post_init__(self):
        L = _abi.lib()
        rep = _abi.replica_array(self.desc.replicas)
        if self.packed:
            g0, g1 = C.c_int64(), C.c_int64()
            _abi.check(L.nbbgpu_plan_packed_partition(rep, self.desc.k, self.desc.s, self.level,
                                                      self.tile_level, self.rank, self.nranks,
                                                      C.byref(g0), C.byref(g1)))
            self.lo, self.hi = g0.value, g1.value
            for p in range(self.nranks):
                if p == self.rank:
                    continue
                self.recv[p] = _packed_needs(self.desc, self.level, self.tile_level, self.rank,
                                             self.nranks, p)
                self.send[p] = _packed_needs(self.desc, self.level, self.tile_level, p, self.nranks,
                                             self.rank)
            return
        lo, hi = C.c_uint64(), C.c_uint64()
        _abi.check(L.nbbgpu_plan_partition(rep, self.desc.k, self.desc.s, self.level, self.tile_level,
                                           self.rank, self.nranks, C.byref(lo), C.byref(hi)))
        self.lo, self.hi = lo.value, hi.value
        for p in range(self.nranks):
            if p == self.rank:
                continue
            self.recv[p] = _needs(self.desc, self.level, self.tile_level, self.rank, self.nranks, p)
            self.send[p] = _needs(self.desc, self.level, self.tile_level, p, self.nranks, self.rank)

    @property
    def peers(self) -> List[int]:
        return [p for p in sorted(self.recv) if self.recv[p].size or self.send[p].size]

    def halo_bytes(self) -> int:
        return int(sum(v.size for v in self.recv.values())) * self.elem_bytes


def exchange(plan: PartitionPlan, dist, pack: Callable[[int], "object"],
             recv_buffer: Callable[[int, int], "object"], unpack: Callable[[int, "object"], None]):
    """One halo exchange: pack(peer) -> tensor of plan.send[peer].size bytes,
    recv_buffer(peer, n) -> tensor to receive into, unpack(peer, tensor)."""
    ops, recvs = [], {}
    for p in plan.peers:
        if plan.send[p].size:
            ops.append(dist.P2POp(dist.isend, pack(p), p))
        if plan.recv[p].size:
            recvs[p] = recv_buffer(p, int(plan.recv[p].size))
            ops.append(dist.P2POp(dist.irecv, recvs[p], p))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    for p, buf in recvs.items():
        unpack(p, buf)


def wrap_u64_sum(values) -> int:
    return int(sum(int(v) & (2**64 - 1) for v in values)) & (2**64 - 1)


class DistributedSimulation:
    """A GPU Simulation that owns one partition of the compact array and exchanges
    halos with its peers after every step.

    transport="nccl" (production): the library's own NCCL communicator (unique id
      broadcast over torch.distributed); pack kernel -> grouped ncclSend/ncclRecv
      -> unpack kernel are enqueued on the engine stream after each step kernel,
      so K steps run without any host synchronisation.
    transport="p2p" (packed kernel): CUDA IPC mappings of the peers' boundary
      planes over NVLink; each step pushes the words peers need straight into their
      planes with a system-scope arrival counter (no NCCL call per step); the IPC
      handles are all-gathered over torch.distributed once.
    transport="torch": torch.distributed point-to-point on device tensors
      (host_staging=True: through host tensors, so gloo can drive several ranks
      that share one test GPU)."""

    def __init__(self, sim, dist, rank: int, nranks: int, transport: str = "auto",
                 host_staging: bool = False):
        import torch
        self.sim, self.dist, self.rank, self.nranks = sim, dist, rank, nranks
        self.transport = transport
        self.host = host_staging
        h = sim.handle()
        L = _abi.lib()
        _abi.check(L.nbbgpu_partition(h, rank, nranks))
        kern, q = sim.active_kernel()  # partition units of the kernel in use
        self.plan = PartitionPlan(sim.desc, sim.level(), rank, nranks, tile_level=q,
                                  packed=kern == "packed")
        lo, hi = C.c_uint64(), C.c_uint64()
        _abi.check(L.nbbgpu_owned_range(h, C.byref(lo), C.byref(hi)))
        if self.plan.packed:
            cp = packed_info(sim.desc, sim.level(), q)["Cp"]
            assert (lo.value, hi.value) == (self.plan.lo * cp, self.plan.hi * cp), "partition geometry mismatch"
        else:
            assert (lo.value, hi.value) == (self.plan.lo, self.plan.hi), "partition geometry mismatch"
        self.launches_per_exchange = (int(any(self.plan.send[p].size for p in self.plan.peers)) +
                                      int(any(self.plan.recv[p].size for p in self.plan.peers)))
        if transport == "auto":
            # peer-memory pushes for the packed kernel when every rank can map its
            # peers' planes (CUDA IPC + NVLink peer access), else the NCCL transport;
            # every collective below is reached by every rank
            mine = None
            if self.plan.packed:
                try:
                    nb = L.nbbgpu_p2p_handle_bytes()
                    buf = (C.c_uint8 * nb)()
                    _abi.check(L.nbbgpu_p2p_export(h, buf, nb))
                    mine = bytes(buf)
                except Exception:  # noqa: BLE001 -- IPC unavailable on this rank
                    mine = None
            allh = [None] * nranks
            dist.all_gather_object(allh, mine)
            if all(x is not None for x in allh):
                ok = 1
                try:
                    nb = len(allh[0])
                    blob = (C.c_uint8 * (nb * nranks)).from_buffer_copy(b"".join(allh))
                    _abi.check(L.nbbgpu_p2p_attach(h, blob, nb, nranks))
                except Exception:  # noqa: BLE001 -- peer mapping failed
                    ok = 0
                flags = [None] * nranks
                dist.all_gather_object(flags, ok)
                if not all(flags):
                    raise RuntimeError("p2p halo transport could not map every peer; use transport='nccl'")
                dist.barrier()
                self.transport = "p2p"
                self.launches_per_exchange = 1
                return
            self.transport = transport = "nccl"
        if transport == "p2p":
            if not self.plan.packed:
                raise ValueError("the p2p transport needs the packed kernel")
            self._attach_p2p(L, h, dist, rank, nranks)
            self.launches_per_exchange = 1
            return
        if transport == "nccl":
            uid = (C.c_uint8 * 128)()
        if transport == "nccl":
            uid = (C.c_uint8 * 128)()
            if rank == 0:
                _abi.check(L.nbbgpu_nccl_unique_id(uid, 128))
            obj = [bytes(uid)]
            dist.broadcast_object_list(obj, src=0)
            uid = (C.c_uint8 * 128).from_buffer_copy(obj[0])
            _abi.check(L.nbbgpu_comm_init(h, uid, 128))
            return
        dev = torch.device("cuda", sim.options.device)
        self._dtype = torch.int32 if self.plan.packed else torch.uint8
        self._send_bufs, self._recv_bufs = {}, {}
        for p in self.plan.peers:
            s = self.plan.send[p]
            _abi.check(L.nbbgpu_halo_set_sends(h, p, s.ctypes.data if s.size else None, s.size))
            self._send_bufs[p] = torch.empty(max(1, s.size), dtype=self._dtype, device=dev)
            self._recv_bufs[p] = torch.empty(max(1, self.plan.recv[p].size), dtype=self._dtype,
                                             device=dev)
        self.launches_per_exchange = sum(int(self.plan.send[p].size > 0) + int(self.plan.recv[p].size > 0)
                                         for p in self.plan.peers)

    def _attach_p2p(self, L, h, dist, rank: int, nranks: int) -> None:
        """All-gather the ranks' IPC handles (boundary planes + arrival counter) and
        map the peers' into this process (nbbgpu_p2p_export / nbbgpu_p2p_attach)."""
        nb = L.nbbgpu_p2p_handle_bytes()
        mine = (C.c_uint8 * nb)()
        _abi.check(L.nbbgpu_p2p_export(h, mine, nb))
        allh = [None] * nranks
        dist.all_gather_object(allh, bytes(mine))
        blob = (C.c_uint8 * (nb * nranks)).from_buffer_copy(b"".join(allh))
        _abi.check(L.nbbgpu_p2p_attach(h, blob, nb, nranks))
        dist.barrier()

    def exchange(self) -> None:
        """torch transport only (the nccl transport exchanges inside every step)."""
        import torch
        if self.transport in ("nccl", "p2p"):
            return
        L, h = _abi.lib(), self.sim.handle()

        def pack(p):
            n = int(self.plan.send[p].size)
            _abi.check(L.nbbgpu_halo_pack(h, p, C.c_void_p(self._send_bufs[p].data_ptr())))
            return self._send_bufs[p][:n].cpu() if self.host else self._send_bufs[p][:n]

        def recv_buffer(p, n):
            return torch.empty(n, dtype=self._dtype) if self.host else self._recv_bufs[p][:n]

        def unpack(p, buf):
            if self.host:
                self._recv_bufs[p][:buf.numel()].copy_(buf)
            torch.cuda.current_stream().synchronize()
            _abi.check(L.nbbgpu_halo_unpack(h, p, C.c_void_p(self._recv_bufs[p].data_ptr())))

        exchange(self.plan, self.dist, pack, recv_buffer, unpack)

    def step(self, rule, nsteps: int = 1) -> None:
        if self.transport in ("nccl", "p2p"):
            self.sim.step(rule, nsteps)
            return
        for _ in range(nsteps):
            self.sim.step(rule)
            self.exchange()

    def step_timed(self, rule, nsteps: int) -> float:
        """Device ms of nsteps steps (step kernels + halo exchanges, one event pair)."""
        if self.transport in ("nccl", "p2p"):
            return self.sim.step_timed(rule, nsteps)
        ms = 0.0
        for _ in range(nsteps):
            ms += self.sim.step_timed(rule, 1)
            self.exchange()
        return ms

    def step_profiled(self, rule, nsteps: int):
        """(total device ms, device ms of the main step kernels, engine kernel launches)."""
        if self.transport in ("nccl", "p2p"):
            return self.sim.step_profiled(rule, nsteps)
        tot = main = 0.0
        launches = 0
        for _ in range(nsteps):
            t, m, n = self.sim.step_profiled(rule, 1)
            tot, main, launches = tot + t, main + m, launches + n + self.launches_per_exchange
            self.exchange()
        return tot, main, launches

    def owned_cells(self) -> int:
        """Compact cells this rank updates per step."""
        if not self.plan.packed:
            return self.plan.hi - self.plan.lo
        info = packed_info(self.sim.desc, self.sim.level(), self.plan.tile_level)
        tiles = min(self.plan.hi * 32, info["T"]) - self.plan.lo * 32
        return tiles * info["C"]

    def state_hash(self) -> int:
        import torch
        v = C.c_uint64()
        _abi.check(_abi.lib().nbbgpu_state_hash_owned(self.sim.handle(), C.byref(v)))
        on_host = self.host or self.dist.get_backend() == "gloo"
        t = torch.tensor([v.value & 0xFFFFFFFF, v.value >> 32], dtype=torch.int64,
                         device="cpu" if on_host else torch.device("cuda", self.sim.options.device))
        parts = [torch.zeros_like(t) for _ in range(self.nranks)]
        self.dist.all_gather(parts, t)
        return wrap_u64_sum(int(q[0]) | (int(q[1]) << 32) for q in parts)


class MultiGpuSimulation:
    """Simulation(..., SimOptions(gpus=N)): ONE process drives N packed partitions,
    one per device (SURVEY.md 8b "one host thread drives all GPUs"; 8e).  Rank i
    owns groups [g0, g1) of the packed layout on devices[i]; the peer-memory
    transport is attached in-process (nbbgpu_p2p_attach_local: the peers' boundary
    planes are device pointers over NVLink, each step pushes the words a peer needs
    and bumps its arrival counter).  step() enqueues every rank's steps (interleaved in
    chunks of 16, so no rank waits on a peer that is not queued yet) and then
    synchronises; ranks
    sharing a device (tests on one GPU) step one at a time instead, since a spinning
    kernel could then starve its peer of SMs.  Same methods as Simulation."""

    def __init__(self, desc: FractalDescriptor, level: int, backend, options):
        from dataclasses import replace
        from .simulation import Simulation
        from .stencil import Backend
        if backend != Backend.GpuCompact or options.block_size > 0:
            raise OutOfDomain("gpus > 1 applies to the linear compact backend")
        n = int(options.gpus)
        devices = list(options.devices) if options.devices is not None else list(range(n))
        if len(devices) != n:
            raise OutOfDomain("SimOptions.devices must list one device per gpu")
        self.desc, self._level, self.options = desc, level, options
        self.devices = devices
        self.shared_device = len(set(devices)) < n
        self.ranks = []
        L = _abi.lib()
        for r in range(n):
            o = replace(options, gpus=1, devices=None, device=devices[r], kernel="packed")
            sim = Simulation(desc, level, backend, o)
            _abi.check(L.nbbgpu_partition(sim.handle(), r, n))
            self.ranks.append(sim)
        arr = (C.c_void_p * n)(*[s.handle().value for s in self.ranks])
        _abi.check(L.nbbgpu_p2p_attach_local(arr, n))
        q = self.ranks[0].active_kernel()[1]
        self.plans = [PartitionPlan(desc, level, r, n, tile_level=q, packed=True) for r in range(n)]
        self._front_cache = None

    # -- lifetime ---------------------------------------------------------------
    def close(self) -> None:
        for s in getattr(self, "ranks", []):
            s.close()
        self.ranks = []

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- geometry -----------------------------------------------------------------
    def level(self) -> int:
        return self._level

    def side(self) -> int:
        return self.ranks[0].side()

    def compact_dims(self):
        return self.ranks[0].compact_dims()

    def iteration(self) -> int:
        return self.ranks[0].iteration()

    def stored_cells(self) -> int:
        return self.ranks[0].stored_cells()

    def peak_bytes(self) -> int:
        return sum(s.peak_bytes() for s in self.ranks)

    def active_kernel(self):
        return self.ranks[0].active_kernel()

    # -- state --------------------------------------------------------------------
    def seed_random(self, seed: int, density: float) -> None:
        self._front_cache = None
        for s in self.ranks:
            s.seed_random(seed, density)

    def step(self, rule: StencilRule, nsteps: int = 1) -> None:
        self._front_cache = None
        for s in self.ranks:
            s._front_cache = None  # stepped below through the C ABI directly
        L = _abi.lib()
        args = (rule.birth & 0xFFFF, rule.survive & 0xFFFF, int(rule.neighborhood == Neighborhood.Moore))
        # distinct devices: chunks of 16 steps per rank, interleaved across ranks (a
        # rank's queue never fills while a peer it waits on is not yet enqueued, and
        # the host issues one call per 16 steps); shared device: one step at a time
        chunk = 1 if self.shared_device else 16
        left = int(nsteps)
        while left > 0:
            k = min(chunk, left)
            for s in self.ranks:
                _abi.check(L.nbbgpu_step_async(s.handle(), *args, k))
                if self.shared_device:
                    _abi.check(L.nbbgpu_synchronize(s.handle()))
            left -= k
        for s in self.ranks:
            _abi.check(L.nbbgpu_synchronize(s.handle()))

    def step_timed(self, rule: StencilRule, nsteps: int) -> float:
        """Wall-clock ms of nsteps on all ranks (enqueue + synchronise)."""
        for s in self.ranks:
            _abi.check(_abi.lib().nbbgpu_synchronize(s.handle()))
        t0 = time.perf_counter()
        self.step(rule, nsteps)
        return (time.perf_counter() - t0) * 1e3

    def state_hash(self) -> int:
        parts = []
        for s in self.ranks:
            v = C.c_uint64()
            _abi.check(_abi.lib().nbbgpu_state_hash_owned(s.handle(), C.byref(v)))
            parts.append(v.value)
        return wrap_u64_sum(parts)

    def front(self):
        if self._front_cache is None:
            g = None
            for s, plan in zip(self.ranks, self.plans):
                f = s.front()
                if g is None:
                    g = f.data.copy()
                m = plan.owned_cell_mask()
                g[m] = f.data[m]
            f0 = self.ranks[0].front()
            self._front_cache = type(f0)(f0.layout, g, f0.width, f0.height, f0.side)
        return self._front_cache

    def upload(self, data: np.ndarray) -> None:
        self._front_cache = None
        for s in self.ranks:
            s.upload(data)

    def cell(self, e) -> int:
        x, y = int(e[0]), int(e[1])
        side = self.side()
        if not (0 <= x < side and 0 <= y < side):
            return self.ranks[0].cell(e)  # the reference's out-of-domain behaviour
        comp, _ = self.ranks[0].nu_batch(np.array([[x, y]], dtype=np.int32))
        cx, cy = int(comp[0][0]), int(comp[0][1])
        if cx < 0 or cy < 0:
            return 0  # not a fractal cell
        w, _ = self.compact_dims()
        return int(self.front().data[cy * w + cx])

    def set_cell(self, e, state: int) -> None:
        self._front_cache = None
        for s in self.ranks:
            s.set_cell(e, state)
