import time, sys
sys.path.insert(0, '/root/repo')
from paper_2110_12952_b200 import Simulation, SimOptions, Backend, builtin_descriptor, conway_rule
from paper_2110_12952_b200 import _abi
import ctypes as C
T = builtin_descriptor("sierpinski-triangle"); Cp = builtin_descriptor("sierpinski-carpet")
for d, r in ((T, 16), (Cp, 9), (T, 18), (T, 14)):
    s = Simulation(d, r, Backend.GpuCompact, SimOptions(kernel="packed", memory_cap=1 << 40))
    s.seed_random(1, 0.5); s.step(conway_rule(), 20)
    K = 1000
    t0 = time.perf_counter(); ms = s.step_timed(conway_rule(), K); wall = time.perf_counter() - t0
    # enqueue-only: async steps then sync
    L = _abi.lib()
    t0 = time.perf_counter()
    _abi.check(L.nbbgpu_step_async(s.handle(), 0x8, 0xC, 1, K))
    t1 = time.perf_counter()
    _abi.check(L.nbbgpu_synchronize(s.handle()))
    t2 = time.perf_counter()
    print(f"{d.name} r={r}: device {ms/K*1e3:.2f} us/step, wall {wall/K*1e6:.2f} us/step, enqueue {(t1-t0)/K*1e6:.2f} us/step, total {(t2-t0)/K*1e6:.2f}")
    s.close()
