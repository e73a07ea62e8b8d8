"""Host<->device conversion timing at T r=20: nbbgpu_upload / nbbgpu_download from / into
pinned host memory vs a plain torch pinned copy of the same bytes."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_12952_b200 import Backend, SimOptions, Simulation, builtin_descriptor, _abi  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 20
T = builtin_descriptor("sierpinski-triangle")
sim = Simulation(T, level, Backend.GpuCompact, SimOptions(memory_cap=1 << 42))
sim.seed_random(42, 0.5)
n = 3 ** level
host = torch.empty(n, dtype=torch.uint8).pin_memory()
L = _abi.lib()
for rep in range(3):
    t0 = time.perf_counter()
    _abi.check(L.nbbgpu_download(sim.handle(), C.c_void_p(host.data_ptr()), n))
    t1 = time.perf_counter()
    _abi.check(L.nbbgpu_upload(sim.handle(), C.c_void_p(host.data_ptr()), n))
    t2 = time.perf_counter()
    print(f"download {n / (t1 - t0) / 1e9:.1f} GB/s  upload {n / (t2 - t1) / 1e9:.1f} GB/s", flush=True)
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev.copy_(host, non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    host.copy_(dev, non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"torch pinned H2D {n / (t1 - t0) / 1e9:.1f} GB/s  D2H {n / (t2 - t1) / 1e9:.1f} GB/s", flush=True)
