import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
from paper_2110_12952_b200 import *
T = builtin_descriptor("sierpinski-triangle")
for r, n in [(20, 1 << 20), (20, 1 << 26), (18, 1 << 26)]:
    sim = Simulation(T, r, Backend.GpuCompact, SimOptions(memory_cap=1 << 42))
    w, h = sim.compact_dims()
    g = torch.Generator(device="cuda").manual_seed(1)
    comp = torch.stack([torch.randint(0, w, (n,), device="cuda", generator=g),
                        torch.randint(0, h, (n,), device="cuda", generator=g)], 1).to(torch.int32).contiguous()
    emb = torch.empty_like(comp); back = torch.empty_like(comp); torch.cuda.synchronize()
    sim.lambda_batch_device(comp.data_ptr(), emb.data_ptr(), n, "digit")
    sim.nu_batch_device(emb.data_ptr(), back.data_ptr(), n, "digit")
    bad = (back != comp).any(1).nonzero().flatten()
    print(r, n, "bad", bad.numel(), comp[bad[:3]].tolist() if bad.numel() else "", emb[bad[:3]].tolist() if bad.numel() else "", back[bad[:3]].tolist() if bad.numel() else "")
    # host path on the first bad ones
    if bad.numel():
        c = comp[bad[:3]].cpu().numpy()
        e2, _ = sim.lambda_batch(c); b2, _ = sim.nu_batch(e2)
        print(" host-path", e2.tolist(), b2.tolist())
    sim.close(); del comp, emb, back; torch.cuda.empty_cache()
for r in range(8, 17, 1):
    for kern in ("tiled", "naive"):
        sim = Simulation(T, r, Backend.GpuCompact, SimOptions(memory_cap=1 << 42, kernel=kern))
        sim.seed_random(1, 0.5); sim.step(conway_rule(), 3)
        ms = sim.step_timed(conway_rule(), 50)
        print("r", r, kern, "%.4f ms" % (ms / 50))
        sim.close()
