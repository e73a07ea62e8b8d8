"""Drives the batched lambda / nu map kernels (digit loop, mma.sync and tcgen05 tensor cores) and the
paper's per-cell step with both map variants, for ncu (T r=16 / r=20)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_12952_b200 import (Backend, SimOptions, Simulation, builtin_descriptor,  # noqa: E402
                                   conway_rule)

T = builtin_descriptor("sierpinski-triangle")
n = 1 << 24
sim = Simulation(T, 20, Backend.GpuCompact, SimOptions(memory_cap=1 << 42))
w, h = sim.compact_dims()
g = torch.Generator(device="cuda").manual_seed(1)
comp = torch.stack([torch.randint(0, w, (n,), device="cuda", generator=g),
                    torch.randint(0, h, (n,), device="cuda", generator=g)], 1).to(torch.int32).contiguous()
emb = torch.empty_like(comp)
back = torch.empty_like(comp)
torch.cuda.synchronize()
for variant in ("digit", "mma", "tc05"):
    sim.lambda_batch_device(comp.data_ptr(), emb.data_ptr(), n, variant)  # warm
    t_l = sim.lambda_batch_device(comp.data_ptr(), emb.data_ptr(), n, variant)
    t_n = sim.nu_batch_device(emb.data_ptr(), back.data_ptr(), n, variant)
    torch.cuda.synchronize()
    print(variant, f"lambda {n / t_l / 1e6:.2f} Gmaps/s, nu {n / t_n / 1e6:.2f} Gmaps/s",
          "exact" if torch.equal(back, comp) else "MISMATCH")
sim.close()
for variant in ("digit", "mma"):
    s = Simulation(T, 16, Backend.GpuCompact, SimOptions(kernel="naive", map_variant=variant))
    s.seed_random(42, 0.5)
    ms = s.step_timed(conway_rule(), 2) / 2
    print("naive step", variant, f"{ms:.3f} ms/step")
    s.close()
