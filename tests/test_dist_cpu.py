"""Host logic of the y-slab decomposition on CPU, world_size 2 over gloo (no GPU): slab layout,
particle partition, the NCCL unique-id handshake, reductions, and bench.py's max-over-ranks."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        from paper_2106_12485_b200 import dist as zd
        cfg = synth.config("C1", nx=16, ny=12)
        p = synth.species_particles(cfg, 0)
        mine = zd.partition(p, cfg["ny"], world, rank)
        y0, n = zd.slab_layout(cfg["ny"], world, rank)
        assert np.all((mine["iy"] >= y0) & (mine["iy"] < y0 + n))
        total = zd.reduce_sum([float(len(mine["ix"]))])[0]
        ids = [None] * world
        dist.all_gather_object(ids, mine["id"].tolist())
        uid = zd.nccl_id_broadcast()
        uids = [None] * world
        dist.all_gather_object(uids, uid)
        mx = zd.reduce_max(float(rank + 1))
        out[rank] = (total, sorted(sum(ids, [])) == sorted(p["id"].tolist()), uids[0] == uids[1] and len(uid) == 128,
                     mx, len(set(ids[0]) & set(ids[1])))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_slab_helpers():
    world = 2
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        total, complete, same_uid, mx, overlap = out[r]
        assert total == 16 * 12 * 16
        assert complete and same_uid and overlap == 0
        assert mx == 2.0


def test_slab_layout_validation():
    from paper_2106_12485_b200 import dist as zd
    assert zd.slab_layout(8192, 8, 3) == (3072, 1024)
    with pytest.raises(ValueError):
        zd.slab_layout(10, 4, 0)
    with pytest.raises(ValueError):
        zd.slab_layout(6, 4, 0)


def test_bench_spawns_one_rank_per_gpu():
    """`bench.py --gpus 2` without a launcher re-runs itself under torch.distributed.run (two
    ranks, rendezvous on 127.0.0.1); with the reference arm (CPU only) rank 0 prints the single
    JSON line with n_gpus = 2 and the other rank exits cleanly.  A launcher whose WORLD_SIZE
    disagrees with --gpus is an error, not a silent 1-GPU run."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0", "--cpu-cells", "64"], capture_output=True, text=True,
                       env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["impl"] == "reference"
    bad = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--gpus", "4",
                          "--steps", "1", "--warmup", "0", "--cpu-cells", "64"], capture_output=True, text=True,
                         env=dict(env, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0"), timeout=600)
    assert bad.returncode != 0 and "WORLD_SIZE" in bad.stderr
