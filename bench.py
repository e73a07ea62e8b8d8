#!/usr/bin/env python3
"""bench.py -- compact cell-updates/s of the B200 compact-fractal stencil engine.

Workload (config.workload): Sierpinski triangle K(n,3,2) at r=20 (3^20 = 3.49e9
compact cells, n = 2^20: the bounding box cannot exist), seed 42, density 0.5,
B3/S23 Moore -- BASELINE.json configs[3], the north-star target; N GPUs split the
compact array into contiguous tile-row ranges with a per-step NVLink halo
exchange (NCCL send/recv via torch.distributed), so scaling is strong.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Timing: W untimed steps, then K steps bracketed by barrier + synchronize, timed
with CUDA events on the engine's stream, max over ranks.  The packed state (0.44 GB
per buffer, 0.87 GB read + written per step) is 7x the 126 MB L2, so no flush is
needed between steps.

One JSON line on rank 0 (see DESIGN.md "Measurement" for every field).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "compact cell-updates/sec (Sierpinski r=16/20) at 1/2/4/8 B200; % HBM roofline"
UNIT = "cell-updates/s"
LEVEL = 20
SEED, DENSITY = 42, 0.5
BIRTH, SURVIVE = 0x8, 0xC  # B3/S23
BYTES_PER_UPDATE = 2       # read own state byte + write next-state byte
PACKED_BYTES_PER_UPDATE = 0.25  # packed model: read own state bit + write next-state bit


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    """dram bytes per launch of the step kernel from the committed ncu --set full capture."""
    path = os.path.join(ROOT, "profiles", "ncu_step_kernel.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d.get("dram_bytes_per_launch"), d
    except Exception:
        return None, None


def gpu_numa_affinity(device: int):
    """Restrict this process to the CPUs NVML reports as local to the GPU; returns
    the previous affinity (None when NVML or the call is unavailable)."""
    try:
        import pynvml as n
        n.nvmlInit()
        hdl = n.nvmlDeviceGetHandleByIndex(device)
        words = n.nvmlDeviceGetCpuAffinity(hdl, (os.cpu_count() + 63) // 64)
        cpus = {64 * i + b for i, w in enumerate(words) for b in range(64) if (w >> b) & 1}
        old = os.sched_getaffinity(0)
        cpus &= old
        if not cpus:
            return None
        os.sched_setaffinity(0, cpus)
        return old
    except Exception:
        return None


class ClockSampler:
    """SM clocks + clock-event (throttle) reasons sampled during the timed region, in
    process through NVML (pynvml): no nvidia-smi process is spawned next to the
    timed kernels.  Falls back to nvidia-smi when pynvml is unavailable."""

    # nvmlClocksEventReason* bits
    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, device):
        self.device = device
        self.rows = []  # (sm_mhz, max_mhz, reason_bits)
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[device]) if vis and vis.split(",")[device].strip().isdigit() else device
            self._h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self._nvml = pynvml
        except Exception:
            self._nvml = None

    def _sample(self):
        if self._nvml is not None:
            n = self._nvml
            try:
                reasons = n.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            except Exception:
                reasons = n.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
            self.rows.append((float(n.nvmlDeviceGetClockInfo(self._h, n.NVML_CLOCK_SM)),
                              float(n.nvmlDeviceGetMaxClockInfo(self._h, n.NVML_CLOCK_SM)), int(reasons)))
            return
        fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                  "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={fields}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
        if out.returncode == 0 and out.stdout.strip():
            c = [x.strip() for x in out.stdout.strip().split(",")]
            bits = sum(v for (name, v), f in zip(self.REASONS.items(), c[2:6]) if f.lower() == "active")
            self.rows.append((float(c[0]), float(c[1]), bits))

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                return
            self._stop.wait(0.01 if self._nvml is not None else 0.2)

    def start(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def stop(self):
        try:
            self._sample()  # one sample at the end of the region too
        except Exception:
            pass
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock query unavailable"]}
        sm = sorted(r[0] for r in self.rows)
        reasons = sorted({name for r in self.rows for name, bit in self.REASONS.items() if r[2] & bit})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(r[1] for r in self.rows), "reasons": reasons,
                "samples": len(self.rows), "source": "nvml" if self._nvml is not None else "nvidia-smi"}


def _device_uuid(device):
    """Physical identity of a CUDA device (ranks sharing one GPU count once)."""
    import torch
    props = torch.cuda.get_device_properties(device)
    uuid = getattr(props, "uuid", None)
    if uuid is None:
        return str(device)
    return bytes(uuid.bytes).hex() if hasattr(uuid, "bytes") else str(uuid)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return ws, rank, local


# ---------------------------------------------------------------------------
# CPU baseline: the reference's own compact step (oracle/_ref) on a bounded sample
# ---------------------------------------------------------------------------
def workload_config(level):
    """The workload (identical for both arms: the driver compares the config dicts);
    how each arm runs it goes under "engine"."""
    cells = 3 ** level
    return {"workload": f"sierpinski-triangle K(2^{level},3,2) r={level} compact, B3/S23 Moore "
                        "(BASELINE.json configs[3]; north-star target)",
            "level": level, "compact_cells": cells, "seed": SEED, "density": DENSITY,
            "l2": (f"inputs larger than L2 ({cells / 1e9:.2f} GB of reference bytes; "
                   f"{(cells + 7) // 8 / 1e9:.2f} GB per packed buffer vs 126 MB L2): no flush")}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_reference_sample(level, cells_target_s=1.0, steps=1, warmup=0, threads=None, full_step=True,
                         single_thread_s=3.0):
    """The reference's own compact step (oracle/_ref: the unmodified proj/src sources,
    -O3 -DNDEBUG like its CMake Release build) on the box's host cores, on the
    reference protocol of bench.cpp:28-59 (full Simulation::step calls,
    stencil.cpp:262-289, workers = all host threads) where it fits the time budget:

      * the whole level-`level` state is seeded (seed 42, density 0.5; the shim's
        threaded seeding writes exactly seed_random's values);
      * `full_step`: one full Simulation::step with workers = nproc (parallel_for);
      * `steps` bounded samples: Simulation::step_compact_linear over a contiguous
        range of ~cells_target_s seconds, split across all threads like parallel_for;
      * a workers = 1 sample of ~single_thread_s seconds.

    Returns a dict; `value` is the full-step rate when measured, else the sample rate."""
    import oracle
    from paper_2110_12952_b200.descriptor import builtin_descriptor
    threads = threads or os.cpu_count() or 1
    T = builtin_descriptor("sierpinski-triangle")
    kind = "reference" if oracle.ref_available() else "port"
    total = 3 ** level
    out = {"unit": UNIT, "cores": threads, "kind": kind, "cpu_model": cpu_model(),
           "host_threads": os.cpu_count()}
    if kind == "reference":
        sim = oracle.RefSim(T.replicas, 3, 2, level, backend="compact", workers=threads,
                            memory_cap=1 << 40)
        t0 = time.perf_counter()
        sim.parallel_seed(SEED, DENSITY, threads)
        out["seed_s"] = time.perf_counter() - t0
        # calibrate: ~4e6 cells/s/thread on the reference; aim for cells_target_s per sample
        n = int(min(total, max(threads * 1e5, 4e6 * threads * cells_target_s)))
        i0 = (total - n) // 2
        for _ in range(warmup):
            sim.sample_step(BIRTH, SURVIVE, True, i0, i0 + n, threads)
        t0 = time.perf_counter()
        for _ in range(steps):
            sim.sample_step(BIRTH, SURVIVE, True, i0, i0 + n, threads)
        dt = (time.perf_counter() - t0) / max(1, steps)
        out["sample_value"] = n / dt
        out["seconds_per_sample"] = dt
        n1 = int(min(total, 4e6 * single_thread_s))
        t0 = time.perf_counter()
        sim.sample_step(BIRTH, SURVIVE, True, i0, i0 + n1, 1)
        out["workers1_value"] = n1 / (time.perf_counter() - t0)
        desc = (f"T r={level}, whole state seeded; {steps} sample(s) of Simulation::step_compact_linear "
                f"over {n} contiguous compact cells (of {total}) on {threads} std::threads "
                f"({out['sample_value']:.3e}/s); workers=1 over {n1} cells ({out['workers1_value']:.3e}/s)")
        if full_step:
            t0 = time.perf_counter()
            sim.step(BIRTH, SURVIVE, True, 1)
            dtf = time.perf_counter() - t0
            out["full_step_s"] = dtf
            out["full_step_value"] = total / dtf
            desc = (f"T r={level}: 1 full Simulation::step (workers={threads}, parallel_for, bench.cpp protocol) "
                    f"{dtf:.1f} s = {total / dtf:.3e}/s; " + desc)
        out["value"] = out.get("full_step_value", out["sample_value"])
        out["sample"] = desc + f"; CPU: {out['cpu_model']}"
        del sim
    else:
        o = oracle.Oracle(T.replicas, 3, 2, min(level, 16))
        o.seed(SEED, DENSITY)
        n = o.w * o.h
        t0 = time.perf_counter()
        for _ in range(steps):
            o.step(BIRTH, SURVIVE, True, threads=threads)
        dt = (time.perf_counter() - t0) / steps
        out.update({"value": n / dt, "seconds_per_sample": dt,
                    "sample": f"oracle port, T r={min(level, 16)} full steps; CPU: {out['cpu_model']}"})
    return out


CPU_KEYS = ("value", "unit", "cores", "kind", "sample", "cpu_model", "host_threads", "full_step_s",
            "full_step_value", "sample_value", "workers1_value")


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    steps, warmup = args.steps, args.warmup
    # each step = one bounded sample sized so the whole run stays within minutes
    budget = max(0.3, min(2.0, 150.0 / max(1, steps + warmup)))
    res = cpu_reference_sample(args.level, cells_target_s=budget, steps=steps, warmup=warmup,
                               full_step=not args.no_full_step)
    # the line's value: the per-step samples (each step = one bounded sample of the
    # workload, as the reference arm requires); the full step is reported beside it
    value = res.get("sample_value", res["value"])
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": steps, "warmup": warmup, "ms_per_step": res["seconds_per_sample"] * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (seed 42, density 0.5)", "impl": "reference",
            "config": workload_config(args.level),
            "engine": {"impl": "oracle/_ref: the unmodified reference sources (-O3 -DNDEBUG)",
                       "parallelism": f"{res['cores']} host threads (parallel_for split)"},
            "cpu_baseline": dict({k: res[k] for k in CPU_KEYS if k in res}, value=value),
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    from paper_2110_12952_b200 import (Backend, SimOptions, Simulation, builtin_descriptor,
                                       conway_rule, _abi)
    ws, rank, local = dist_env()
    dist = None
    device = (local if ws > 1 else 0) if args.device is None else args.device
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(device)
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", device))
        else:  # test knob: several ranks sharing one GPU, halo staged through the host
            dist.init_process_group("gloo")
    T = builtin_descriptor("sierpinski-triangle")
    rule = conway_rule()
    L = _abi.lib()
    sim = Simulation(T, args.level, Backend.GpuCompact, SimOptions(memory_cap=1 << 40, device=device))
    h = sim.handle()
    cells = 3 ** args.level
    kern, q = sim.active_kernel()
    sim.seed_random(SEED, DENSITY)

    # ---- partition + halo plan (host-only lists; no communication needed) ----
    dsim = None
    if ws > 1:
        from paper_2110_12952_b200.distributed import DistributedSimulation
        if args.transport in ("p2p", "auto"):
            dsim = DistributedSimulation(sim, dist, rank, ws, transport=args.transport)
        elif args.dist_backend == "nccl" and args.transport == "nccl":
            dsim = DistributedSimulation(sim, dist, rank, ws, transport="nccl")
        elif args.dist_backend == "nccl":
            dsim = DistributedSimulation(sim, dist, rank, ws, transport="torch")
        else:
            dsim = DistributedSimulation(sim, dist, rank, ws, transport="torch", host_staging=True)
        owned = dsim.owned_cells()
        devs = [None] * ws
        dist.all_gather_object(devs, _device_uuid(device))
        n = len(set(devs))  # GPUs that actually stepped (ranks sharing a device count once)
    else:
        owned = cells
        n = 1

    def exchange():
        if dsim is not None:
            dsim.exchange()  # no-op for the in-library nccl transport

    def barrier():
        torch.cuda.synchronize(device)
        if dist is not None:
            dist.barrier()

    # ---- warmup --------------------------------------------------------------
    for _ in range(args.warmup):
        sim.step(rule)
        exchange()

    # ---- timed: device-resident state, K steps ---------------------------------
    stream = C.c_void_p()
    _abi.check(L.nbbgpu_stream(h, C.byref(stream)))
    ext = torch.cuda.ExternalStream(stream.value, device=f"cuda:{device}")
    clocks = ClockSampler(device)
    barrier()
    clocks.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    n0 = C.c_uint64()
    _abi.check(L.nbbgpu_launch_count(h, C.byref(n0)))
    t_wall = time.perf_counter()
    # K steps back to back on the engine stream (packed: halo-words kernel + step
    # kernel per step; N > 1 adds the peer push or the NCCL exchange on-stream).
    # The library records its CUDA events on the engine stream right around the K
    # launches (nbbgpu_step_timed); torch events around the ctypes call would also
    # count the host's call/return latency while the stream idles (~3 us/step at K=20)
    if ws == 1 or dsim.transport in ("nccl", "p2p"):
        step_ms = sim.step_timed(rule, args.steps)
    else:
        ev0.record(ext)
        dsim.step(rule, args.steps)
        ev1.record(ext)
    barrier()
    t_wall = time.perf_counter() - t_wall
    clk = clocks.stop()
    if not (ws == 1 or dsim.transport in ("nccl", "p2p")):
        step_ms = ev0.elapsed_time(ev1)
    n1 = C.c_uint64()
    _abi.check(L.nbbgpu_launch_count(h, C.byref(n1)))
    launches = n1.value - n0.value
    if dsim is not None and dsim.transport == "torch":
        launches += args.steps * dsim.launches_per_exchange
    # second pass of K steps with CUDA events around every main step kernel: its own
    # average duration for the roofline (per-kernel events add gaps, so the headline
    # value above is timed without them)
    barrier()
    if ws == 1:
        _, kernel_ms, _ = sim.step_profiled(rule, args.steps)
    else:
        _, kernel_ms, _ = dsim.step_profiled(rule, args.steps)
    barrier()
    if dist is not None:
        tt = torch.tensor([step_ms, kernel_ms], dtype=torch.float64,
                          device=f"cuda:{device}" if args.dist_backend == "nccl" else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        step_ms, kernel_ms = float(tt[0]), float(tt[1])
    ms_per_step = step_ms / args.steps
    value = cells * args.steps / (step_ms / 1e3)

    # ---- parity sanity: hash of the final state equals across GPU counts -------
    final_hash = dsim.state_hash() if dsim is not None else sim.state_hash()

    # ---- e2e through the public API with host buffers ----------------------------
    # upload the initial state from pinned host memory, K synchronous
    # Simulation.step calls (one C-ABI call each, like nbb::Simulation::step),
    # download the final state into pinned host memory.  All inside the region.
    e2e = None
    if not args.no_e2e:
        # host buffers and the driving thread on the GPU's own NUMA node (NVML CPU
        # affinity): pinned pages are placed by first touch, and PCIe DMA to a remote
        # node's memory is slower and noisier; the previous affinity is restored after
        old_aff = gpu_numa_affinity(device)
        host_in = torch.empty(cells, dtype=torch.uint8).pin_memory()
        host_out = torch.empty(cells, dtype=torch.uint8).pin_memory()
        _abi.check(L.nbbgpu_download(h, C.c_void_p(host_in.data_ptr()), cells))
        reps = []
        for rep in range(6):  # 1 untimed + median of 5 end-to-end runs (host memory behaviour varies)
            barrier()
            t0 = time.perf_counter()
            _abi.check(L.nbbgpu_upload(h, C.c_void_p(host_in.data_ptr()), cells))
            for _ in range(args.steps):
                sim.step(rule)
                exchange()
            _abi.check(L.nbbgpu_download(h, C.c_void_p(host_out.data_ptr()), cells))
            barrier()
            if rep:
                reps.append(time.perf_counter() - t0)
        e2e_s = sorted(reps)[len(reps) // 2]
        if old_aff is not None:
            os.sched_setaffinity(0, old_aff)
        if dist is not None:
            tt = torch.tensor([e2e_s], dtype=torch.float64,
                              device=f"cuda:{device}" if args.dist_backend == "nccl" else "cpu")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_s = float(tt[0])
        e2e = {"value": cells * args.steps / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": cells / args.steps, "d2h_bytes_per_step": cells / args.steps,
               "how": ("upload(pinned host state, reference bytes) + K x nbbgpu_step(1) + download(pinned "
                       "host, reference bytes), wall clock, median of 5 after one untimed run; the bytes<->packed conversion "
                       "runs on the device, pipelined with the DMA copies")}

    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    peak, peak_src = peaks()
    kernel_ms_isolated = kernel_ms / args.steps
    kernel_ms_per_launch = kernel_ms_isolated
    timing = ("CUDA events around every step kernel launch (second pass of K steps; the events "
              "serialise the launches, so each launch is timed without its PDL overlap)")
    if ws == 1 and launches == args.steps:
        # one launch per step (the step kernel gathers its halo words itself): the timed
        # region is exactly K launches of this kernel, so its average launch duration is
        # the timed region / K, PDL overlap of consecutive launches included
        kernel_ms_per_launch = step_ms / args.steps
        timing = ("one launch per step: CUDA events around the K back-to-back launches of the timed "
                  "region on the engine stream / K")
    packed = kern == "packed"
    # algorithmic bytes per launch: packed layout = read + write 1 bit per owned cell
    # (SURVEY.md 8d's packed model); byte layouts = 2 B per owned cell
    bpu = PACKED_BYTES_PER_UPDATE if packed else BYTES_PER_UPDATE
    achieved = bpu * owned / (kernel_ms_per_launch / 1e3) / 1e9
    achieved_2b = BYTES_PER_UPDATE * owned / (kernel_ms_per_launch / 1e3) / 1e9
    traffic, ncu = ncu_traffic()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": "u32 bit-sliced (1 bit per cell, 32 tiles per word)" if packed else "u8",
        "data": "synthetic: seed_random(42, 0.5) generated on the device (rng.hpp cell_alive)",
        "config": workload_config(args.level),
        "engine": {"kernel": f"{kern} (tile level q={q})",
                   "parallelism": (f"partitioned x{ws} over {n} GPU(s), halo transport {dsim.transport}"
                                   if dsim is not None else "single GPU"),
                   "partitions": ws,
                   "state_bytes_per_buffer": (cells + 7) // 8 if packed else cells},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "model": ("packed: 2 bits (read own + write next state, 1 bit each) per compact "
                               "cell-update x owned cells per launch (SURVEY.md 8d packed model)" if packed else
                               "2 B per compact cell-update (SURVEY.md 8d) x owned cells per launch"),
                     "peak_source": peak_src, "kernel_ms_per_launch": kernel_ms_per_launch,
                     "kernel_timing": timing, "kernel_ms_isolated": kernel_ms_isolated,
                     "model_2B": {"achieved": achieved_2b, "frac": achieved_2b / peak,
                                  "note": "the reference's 1 byte per cell (grid.hpp:15); > 1 means the "
                                          "packed layout moves fewer bytes than the byte model assumes"}},
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk,
        "final_state_hash": f"{final_hash:016x}",
        "wall_s": t_wall,
    }
    if ncu:
        line["roofline"]["ncu"] = {k: v for k, v in ncu.items() if k != "dram_bytes_per_launch"}
    if not args.no_cpu_baseline and n == 1:
        try:
            line["cpu_baseline"] = {k: v for k, v in cpu_reference_sample(
                args.level, 2.0, 3, 1, full_step=not args.no_full_step).items() if k in CPU_KEYS}
        except Exception as e:  # reported, not fatal
            line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-full-step", action="store_true",
                    help="skip the full-step CPU measurement (~35 s at r=20 on 16 threads)")
    ap.add_argument("--level", type=int, default=LEVEL, help="triangle level (default 20)")
    ap.add_argument("--device", type=int, default=None, help="test knob: force the CUDA device")
    ap.add_argument("--transport", choices=["auto", "nccl", "p2p", "torch"], default="auto",
                    help="halo transport: auto (default) = peer-memory pushes over NVLink (p2p, CUDA IPC) "
                         "when every rank can map its peers, else the in-library NCCL send/recv on the "
                         "engine stream; torch = torch.distributed point-to-point")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="test knob: gloo lets several ranks share one GPU")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    ws, _, _ = dist_env()
    if ws == 1 and args.gpus > 1:
        return relaunch_distributed(args)
    return run_ours(args)


def relaunch_distributed(args):
    """`python bench.py --gpus N` without torchrun: re-run this script as N ranks
    (one process per GPU) exactly as the driver launches it, so the line always
    measures N devices.  Refuses (exit 2, no line claiming N GPUs) when fewer than N
    devices are visible, unless --device pins every rank to one device (test knob:
    N partitions emulated on one GPU, reported as n_gpus 1, partitions N)."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if args.device is None and have < args.gpus:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} needs {args.gpus} visible GPUs, "
                                                     f"found {have}", "n_gpus": have}), flush=True)
        return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


if __name__ == "__main__":
    sys.exit(main())
