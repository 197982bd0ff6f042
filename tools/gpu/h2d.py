"""Diagnostics: pinned host->device bandwidth, and the time split of zpic_set_particles at C5 scale."""
import time
import torch
import numpy as np
n = 1 << 30   # 4 GiB of float32
h = torch.empty(n, dtype=torch.float32, pin_memory=True)
d = torch.empty(n, dtype=torch.float32, device="cuda")
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    print("H2D pinned 4 GiB: %.1f GB/s" % (4 * 2**30 / (time.perf_counter() - t) / 1e9))
del d, h
import sys, os
sys.path.insert(0, os.getcwd())
import synth, paper_2106_12485_b200 as z
cfg = synth.config("C5")
src = z.Simulation(cfg, inject=True)
p = src.particles(0)
src.close()
pinned = {}
for k, v in p.items():
    t = torch.empty(v.shape, dtype={np.int32: torch.int32, np.float32: torch.float32}[v.dtype.type], pin_memory=True)
    t.numpy()[...] = v
    pinned[k] = t
del p
sim = z.Simulation(cfg, inject=False)
for rep in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    sim.set_particles(0, {k: v.numpy() for k, v in pinned.items()})
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    nb = sum(v.numel() * v.element_size() for v in pinned.values())
    print("set_particles C5: %.3f s, %.1f GB/s of host data" % (dt, nb / dt / 1e9))
