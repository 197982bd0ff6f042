"""The per-GPU cost of one C5 slab (1/8 of C5: 8192 x 1024 cells, 16 ppc) on one B200 under each
halo transport and current variant, as a one-rank ring (every halo kernel of a real rank runs;
the neighbour is the context itself), next to the unsplit periodic domain of the same size:
  unsplit   current_mode 0 (reduction) / 1 (commutative), plain launches and graphs;
  nccl      NCCL send / recv rounds on the comm stream (current_mode 0);
  peer      the library's peer-put / signal / wait kernels, current_mode 0 (reduction rounds)
            and 1 (the slab-edge tiles add their ghost rows into the neighbour's J).
Then an 8-slab loopback group of the whole C5 grid (all slabs serialised on one stream: the sum of
the slabs' kernels) for loopback copies vs PEER, both current modes.
Prints one JSON line per point (CUDA events on the context's stream, after warm-up)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import synth  # noqa: E402
import paper_2106_12485_b200 as z  # noqa: E402
from paper_2106_12485_b200.dist import LoopbackGroup  # noqa: E402


def timed(step, stream, steps=10, warmup=3):
    step(warmup)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    step(steps)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def emit(**kw):
    print(json.dumps(kw), flush=True)


cfg = synth.config("C5")
cfg["ny"] = cfg["ny"] // 8
cfg["name"] += "-slab-of-8"
cases = [("unsplit", 0, True), ("unsplit", 1, True), ("unsplit", 0, False), ("unsplit", 1, False),
         ("nccl", 0, True), ("peer", 0, False), ("peer", 1, False)]
for tr, cm, graphs in cases:
    dist = None
    if tr == "nccl":
        dist = {"rank": 0, "world": 1, "transport": "nccl", "nccl_id": z.zpic.zpic_nccl_unique_id()}
    elif tr == "peer":
        dist = {"rank": 0, "world": 1, "transport": "peer"}
    sim = z.Simulation(cfg, inject=True, dist=dist, current_mode=cm, graphs=graphs)
    n = sim.counters()["particles"]
    ms = timed(sim.step, sim.torch_stream)
    emit(case="ring", config=cfg["name"], transport=tr, current_mode=cm, graphs=graphs, ms_per_step=ms,
         pushes_per_s=n / (ms * 1e-3), launches_per_step=None)
    sim.close()
    del sim
    torch.cuda.empty_cache()

full = synth.config("C5")
for tr in ("loopback", "loopback_peer"):
    for cm in (0, 1):
        g = LoopbackGroup(full, 8, transport=tr, inject=True, current_mode=cm)
        n = g.counters()["particles"]
        ms = timed(g.step, g.stream)
        emit(case="group8", config="C5", transport=tr, current_mode=cm, ms_per_step=ms, pushes_per_s=n / (ms * 1e-3))
        g.close()
        del g
        torch.cuda.empty_cache()
