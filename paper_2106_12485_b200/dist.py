"""Host-side helpers of the y-slab decomposition (the paper's row-band
regions): slab layout, partition of a global particle set by slab, the NCCL
unique-id handshake over torch.distributed, and loopback groups of slab contexts on one GPU.
No physics here: every stage of the step runs in the CUDA library."""
import numpy as np


def slab_layout(ny, world, rank):
    """(y0, ny_local) of `rank`: equal row bands, ny % world == 0, >= 2 rows each."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    if ny % world or ny // world < 2:
        raise ValueError("ny must be a multiple of world with >= 2 rows per slab")
    n = ny // world
    return rank * n, n


def partition(particles, ny, world, rank):
    """The particles of a global set that belong to `rank`'s slab (global iy kept)."""
    y0, n = slab_layout(ny, world, rank)
    m = (particles["iy"] >= y0) & (particles["iy"] < y0 + n)
    return {k: np.ascontiguousarray(v[m]) for k, v in particles.items()}


def slab_rows(field, ny, world, rank):
    """Rows of a global [comp][y][x] field owned by `rank`."""
    y0, n = slab_layout(ny, world, rank)
    return np.ascontiguousarray(field[:, y0:y0 + n, :])


def nccl_id_broadcast(group=None):
    """Rank 0 creates an ncclUniqueId through the library, every rank receives it through
    torch.distributed (any backend, gloo included)."""
    import torch.distributed as dist
    obj = [None]
    if dist.get_rank(group) == 0:
        from .zpic import zpic_nccl_unique_id
        obj[0] = zpic_nccl_unique_id()
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def reduce_sum(values, group=None):
    """Sum a list of floats over the ranks (energies, counts) with torch.distributed."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(values, dtype=torch.float64)
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    dist.all_reduce(t, group=group)
    return t.cpu().tolist()


def reduce_max(value, group=None):
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64)
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


class LoopbackGroup:
    """`world` slab contexts of one decomposition in this process, on one GPU and one stream,
    stepped together (zpic_step_group).  Validates the slab exchange logic on a single GPU."""

    def __init__(self, cfg, world, transport="loopback", **kw):
        """transport: "loopback" (the rounds as device copies between the contexts) or
        "loopback_peer" (the PEER transport's own put / signal / wait kernels)."""
        import torch
        from .zpic import Simulation
        self.stream = torch.cuda.Stream()
        self.sims = [Simulation(cfg, stream=self.stream, dist={"rank": r, "world": world, "transport": transport},
                                **kw) for r in range(world)]
        self.world = world
        self.cfg = cfg

    def set_particles(self, s, p):
        for r, sim in enumerate(self.sims):
            sim.set_particles(s, partition(p, self.cfg["ny"], self.world, r))

    def set_fields(self, which, arr):
        for r, sim in enumerate(self.sims):
            sim.set_fields(which, slab_rows(arr, self.cfg["ny"], self.world, r))

    def step(self, n=1):
        from .zpic import zpic_step_group
        zpic_step_group([s.ctx for s in self.sims], n)

    def fields(self, which):
        return np.concatenate([s.fields(which) for s in self.sims], axis=1)

    def particles(self, s, with_id=False):
        parts = [sim.particles(s, with_id) for sim in self.sims]
        return {k: np.concatenate([p[k] for p in parts]) for k in parts[0]}

    def energy(self):
        its, fes, kes = zip(*[s.energy() for s in self.sims])
        return its[0], float(sum(fes)), [float(sum(k[q] for k in kes)) for q in range(len(kes[0]))]

    def counters(self):
        cs = [s.counters() for s in self.sims]
        return {"particles": sum(c["particles"] for c in cs)}

    def close(self):
        for s in self.sims:
            s.close()
