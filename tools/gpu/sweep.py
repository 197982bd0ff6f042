"""SURVEY.md NEXT-2 on one B200: the paper's decomposition questions (region size, regions per
core; Figs. 4-5) asked of this build.
  1. tile size T (the region analogue) for C5 and the paper's warm plasma (256 ppc);
  2. y-slabs per GPU (loopback contexts on one device, the overdecomposition analogue) for C5.
Prints one JSON line per point: particle pushes/s over `steps` timed steps (CUDA events)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
import synth  # noqa: E402
import paper_2106_12485_b200 as z  # noqa: E402
from paper_2106_12485_b200.dist import LoopbackGroup  # noqa: E402


def timed(step, stream, n_particles, steps=10, warmup=3):
    step(warmup)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    step(steps)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    return ms, n_particles / (ms * 1e-3)


for name in ("C5", "P-WARM"):
    for T in (8, 16, 32):
        cfg = synth.config(name)
        try:
            sim = z.Simulation(cfg, inject=True, tile=T, graphs=False)
        except z.ZpicError as e:
            print(json.dumps({"sweep": "tile", "config": name, "tile": T, "error": str(e)}), flush=True)
            continue
        n = sim.counters()["particles"]
        ms, v = timed(sim.step, sim.torch_stream, n)
        print(json.dumps({"sweep": "tile", "config": name, "tile": T, "ms_per_step": ms, "pushes_per_s": v}), flush=True)
        sim.close()
        torch.cuda.empty_cache()

for k in (1, 2, 4, 8):
    cfg = synth.config("C5")
    if k == 1:
        sim = z.Simulation(cfg, inject=True, tile=16, graphs=False)
        n = sim.counters()["particles"]
        ms, v = timed(sim.step, sim.torch_stream, n)
        sim.close()
    else:
        grp = LoopbackGroup(cfg, k, inject=True, tile=16)
        n = grp.counters()["particles"]
        ms, v = timed(grp.step, grp.stream, n)
        grp.close()
    torch.cuda.empty_cache()
    print(json.dumps({"sweep": "slabs_per_gpu", "config": "C5", "slabs": k, "ms_per_step": ms, "pushes_per_s": v}),
          flush=True)
