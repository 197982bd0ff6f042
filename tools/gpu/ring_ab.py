"""One C5 slab of an 8-GPU split (8192 x 1024) as a one-rank ring, PEER and NCCL transports, vs
the unsplit domain; run under different environment switches by the caller (same-box A/B)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import synth  # noqa: E402
import paper_2106_12485_b200 as z  # noqa: E402

cfg = synth.config("C5")
cfg["ny"] = cfg["ny"] // 8
tag = sys.argv[1] if len(sys.argv) > 1 else ""
for tr, cm in (("unsplit", 0), ("peer", 0), ("peer", 1), ("nccl", 0)):
    dist = None
    if tr == "peer":
        dist = {"rank": 0, "world": 1, "transport": "peer"}
    elif tr == "nccl":
        dist = {"rank": 0, "world": 1, "transport": "nccl", "nccl_id": z.zpic.zpic_nccl_unique_id()}
    sim = z.Simulation(cfg, inject=True, dist=dist, current_mode=cm, graphs=tr != "unsplit" or True)
    sim.step(3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(sim.torch_stream)
    sim.step(12)
    e1.record(sim.torch_stream)
    torch.cuda.synchronize()
    print(json.dumps({"tag": tag, "transport": tr, "current_mode": cm, "ms_per_step": e0.elapsed_time(e1) / 12}),
          flush=True)
    sim.close()
    del sim
    torch.cuda.empty_cache()
