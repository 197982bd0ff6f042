"""Benchmark of the B200 EM-PIC hot path (BASELINE.json metric: particle pushes/s, % of the HBM
roofline).  Contract: `python bench.py --gpus N --steps K --warmup W` prints ONE JSON line on
rank 0.  Workload (N=1): BASELINE.json configs[4] "C5" (8192^2 cells, 4x4 ppc, 1.07e9
particles, uth 0.1, periodic), the configuration the metric and the roofline target are quoted
on.  `--impl reference` times the fp64 oracle (the reference arm of this tier) on the host.

Timing: W untimed warm-up steps, then K steps bracketed by barrier + cuda synchronize, CUDA
events on the library's stream (= torch's current stream), max over ranks.  The particle
store (30 GB) is far larger than the 126 MB L2, so no L2 flush is needed between steps.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "particle pushes/s (push+deposit)"
UNIT = "particles/s"
# algorithmic bytes of the fused push+deposit kernel (K1) per launch:
# 56 B per particle (read + write ix, iy, x, y, ux, uy, uz) + 36 B per cell (E, B read, J write).
K1_BYTES_PER_PARTICLE = 56
K1_BYTES_PER_CELL = 36


def numa_bind(device):
    """Pin this process to the CPUs of the GPU's NUMA node (sysfs local_cpulist of its PCI
    device), so the pinned host buffers of the end-to-end leg are allocated next to the GPU's PCIe
    root.  No-op when the topology is not readable."""
    try:
        bus = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader", "-i", str(device)],
                             capture_output=True, text=True, timeout=20).stdout.strip().lower()
        dom, rest = bus.split(":", 1)
        path = "/sys/bus/pci/devices/%s:%s/local_cpulist" % (dom[-4:], rest)
        cpus = set()
        for part in open(path).read().strip().split(","):
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
        if cpus:
            os.sched_setaffinity(0, cpus)
            return sorted(cpus)
    except Exception:
        pass
    return None


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def launch_ranks(args, argv):
    """`--gpus N` without a launcher: re-run this script under torch.distributed.run, one rank per
    GPU of this node (rendezvous on 127.0.0.1).  Under a launcher WORLD_SIZE must equal --gpus."""
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if world:
        if world != args.gpus:
            sys.exit("bench.py: --gpus %d but WORLD_SIZE=%d" % (args.gpus, world))
        return False
    if args.gpus <= 1:
        return False
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + argv
    sys.exit(subprocess.call(cmd))


def k1_traffic(config, nx, ny):
    """DRAM bytes per K1 launch from the committed ncu capture of the same workload
    (profiles/r2_k1_traffic_c5.json), else None."""
    p = os.path.join(ROOT, "profiles", "r2_k1_traffic_c5.json")
    if config == "C5" and (nx, ny) == (8192, 8192) and os.path.exists(p):
        return json.load(open(p))["per_launch_bytes"]
    return None


def full_count(cfg):
    """Particles of a config's uniform species (nx ny ppc each); None if a species is not uniform."""
    n = 0
    for sp in cfg["species"]:
        if sp.get("profile", "uniform") != "uniform":
            return None
        n += cfg["nx"] * cfg["ny"] * sp["ppc"][0] * sp["ppc"][1]
    return n


def workload_name(name, cfg, n_particles):
    """config.workload: the synth config, its BASELINE.json index if it is one, and its shape."""
    idx = {"C1": 0, "C2": 1, "C3": 2, "C4": 3, "C5": 4}.get(name)
    sp = cfg["species"]
    ppc = "+".join("%dx%d" % tuple(s["ppc"]) for s in sp)
    bc = {0: "periodic", 1: "open", 2: "window"}
    count = "%d particles, " % n_particles if n_particles is not None else ""
    return "%s%s: %dx%d cells, %d species, ppc %s, %sbc x %s / y %s" % (
        cfg["name"], " (BASELINE.json configs[%d])" % idx if idx is not None else " (SURVEY.md NEXT-3)",
        cfg["nx"], cfg["ny"], len(sp), ppc, count, bc[cfg["bc"][0]], bc[cfg["bc"][1]])


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.Q,
                                       "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].strip().replace(".", "").isdigit()]
        pw = [float(r[3]) for r in rows if len(r) >= 9 and r[3].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            if len(r) < 9:
                continue
            for k, nm in enumerate(names):
                if "Active" in r[5 + k] and "Not" not in r[5 + k]:
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(rows),
                "power_w": statistics.median(pw) if pw else None}


def host_info():
    """The host the oracle ran on: logical CPUs and the CPU model."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def cpu_baseline(args):
    """The oracle, as it stands, on a bounded sample of the same workload: the
    physics of the benchmarked config on a cpu_cells^2 periodic patch, `cpu_steps` steps, pinned to
    one host core (sched_setaffinity, the taskset equivalent), repeated `cpu_reps` times; the mean
    and the spread of the repetitions are reported."""
    import synth
    from oracle.sim import from_config
    cfg = synth.config(args.config, nx=args.cpu_cells, ny=args.cpu_cells)
    if any(sp.get("profile", "uniform") != "uniform" for sp in cfg["species"]):
        cfg = synth.config("C5", nx=args.cpu_cells, ny=args.cpu_cells)
    old = os.sched_getaffinity(0)
    core = min(old)
    os.sched_setaffinity(0, {core})
    rates = []
    try:
        for _ in range(args.cpu_reps):
            sim = from_config(cfg)
            n = sum(len(s["ix"]) for s in sim.species)
            t0 = time.perf_counter()
            for _ in range(args.cpu_steps):
                sim.step()
            rates.append(n * args.cpu_steps / (time.perf_counter() - t0))
            del sim
    finally:
        os.sched_setaffinity(0, old)
    return {"value": statistics.mean(rates), "unit": UNIT, "cores": 1, "kind": "oracle", "core": core,
            "std": statistics.pstdev(rates), "repetitions": len(rates),
            "sample": "%s physics on a %dx%d-cell periodic patch (%d particles), %d steps x %d repetitions, fp64 "
                      "serial oracle pinned to core %d" % (cfg["name"], args.cpu_cells, args.cpu_cells, n,
                                                          args.cpu_steps, args.cpu_reps, core),
            **host_info()}


def run_reference(args, world, rank):
    """--impl reference: the oracle (the reference arm of this tier) on the box's host cores."""
    if rank != 0:
        return
    import synth
    from oracle.sim import from_config
    # bound the run to a few minutes: ~3 s per oracle step on a 1024^2 patch, so past 50 steps the
    # patch shrinks with the step count (a multiple of 64 cells per side)
    tot = max(1, args.steps + args.warmup)
    if tot > 50:
        args.cpu_cells = max(64, int(args.cpu_cells * (50.0 / tot) ** 0.5) // 64 * 64)
    cfg = synth.config(args.config, nx=args.cpu_cells, ny=args.cpu_cells)
    sim = from_config(cfg)
    n = sum(len(s["ix"]) for s in sim.species)
    for _ in range(args.warmup):
        sim.step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        sim.step()
    dt = time.perf_counter() - t0
    v = n * args.steps / dt
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": workload_name(args.config, synth.config(args.config), full_count(synth.config(args.config))),
                       "sample": "%s physics on a %dx%d-cell periodic patch, %d particles (the oracle takes ~3 s "
                                 "per step there; the full workload would take hours)" % (args.config, args.cpu_cells,
                                                                                           args.cpu_cells, n)},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": "%dx%d-cell periodic patch of %s, %d particles, %d steps"
                                       % (args.cpu_cells, args.cpu_cells, args.config, n, args.steps),
                             **host_info()},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def e2e_run(args, cfg, torch, z, dist_kw=None, world=1):
    """End to end through the public API with HOST buffers: upload the initial particles from
    pinned host memory (zpic_set_particles), K steps with the energies read back every step,
    and the final E, B fields read back; all inside the timed region (max over ranks)."""
    import numpy as np
    if dist_kw is not None:
        from paper_2106_12485_b200.dist import nccl_id_broadcast
        dist_kw = dict(dist_kw, nccl_id=nccl_id_broadcast())
    import synth
    src = z.Simulation(cfg, inject=True, dist=dist_kw, tile=args.tile, current_precision=args.current_precision)
    host = []
    for s in range(len(cfg["species"])):
        p = src.particles(s)
        pinned = {}
        for k, v in p.items():
            t = torch.empty(v.shape, dtype={np.int32: torch.int32, np.float32: torch.float32}[v.dtype.type],
                            pin_memory=True)
            t.numpy()[...] = v
            pinned[k] = t
        host.append(pinned)
    src.close()
    del p
    laser = synth.laser_fields(cfg) if "laser" in cfg else ()
    if dist_kw is not None:   # a fresh communicator for the second context
        from paper_2106_12485_b200.dist import nccl_id_broadcast
        dist_kw = dict(dist_kw, nccl_id=nccl_id_broadcast())
    sim = z.Simulation(cfg, inject=False, dist=dist_kw, tile=args.tile, current_precision=args.current_precision)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    # pinned host buffers for the read-back fields (allocated outside the timed region, like the inputs)
    y0, nyl = z.zpic.zpic_layout(sim.ctx)
    fout = [torch.empty((3, nyl, cfg["nx"]), dtype=torch.float32, pin_memory=True) for _ in range(2)]
    t0 = time.perf_counter()
    h2d = 0
    for s, hp in enumerate(host):
        sim.set_particles(s, {k: v.numpy() for k, v in hp.items()})
        h2d += sum(v.numel() * v.element_size() for v in hp.values())
    for w, F in enumerate(laser):
        sim.set_fields(w, F)
        h2d += F.nbytes
    t1 = time.perf_counter()
    d2h = 0
    for _ in range(args.steps):
        sim.step(1)
        sim.energy()
        d2h += 8 * (1 + len(cfg["species"]))
    t2 = time.perf_counter()
    for w in (0, 1):
        f = z.zpic.zpic_get_fields(sim.ctx, w, cfg["nx"], nyl, out=fout[w].numpy())
        d2h += f.nbytes
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    dt = t3 - t0
    split = {"upload_s": t1 - t0, "steps_s": t2 - t1, "readback_s": t3 - t2}
    n = sum(v["ix"].numel() for v in host)
    sim.close()
    if world > 1:
        from paper_2106_12485_b200.dist import reduce_max, reduce_sum
        dt = reduce_max(dt)
        n, h2d, d2h = reduce_sum([float(n), float(h2d), float(d2h)])
    return {"value": n * args.steps / dt, "unit": UNIT, "h2d_bytes_per_step": int(h2d / args.steps),
            "d2h_bytes_per_step": int(d2h / args.steps), "seconds": dt, **split,
            "note": "initial particles uploaded from pinned host memory, energies read every step, E and B read "
                    "into pinned memory at the end"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    # default W + K = 50: the whole 50-step C5 workload (BASELINE.json configs[4]); the K1 time
    # grows over the first ~30 steps as the in-tile particle order decays
    ap.add_argument("--steps", type=int, default=47)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--tile", type=int, default=0, help="tile size (0 = the library's auto choice)")
    ap.add_argument("--cpu-cells", type=int, default=512)
    ap.add_argument("--cpu-steps", type=int, default=3)
    ap.add_argument("--cpu-reps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--nx", type=int, default=0, help="override the grid (profiling runs only)")
    ap.add_argument("--ny", type=int, default=0)
    ap.add_argument("--graphs", action="store_true",
                    help="time zpic_step with CUDA-graph replay (no per-kernel events: no roofline / kernel times)")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "peer"],
                    help="y-slab halo rounds at N>1: NCCL send / recv, or the library's peer-put kernels over "
                         "CUDA IPC peer memory (NVLink)")
    ap.add_argument("--current-mode", type=int, default=0, choices=[0, 1],
                    help="0 = tile-block reduction (K4), 1 = commutative global atomics (SURVEY.md NEXT-4)")
    ap.add_argument("--current-precision", default="auto", choices=["auto", "exact"],
                    help="fixed-point tile current: auto (one int32 per node at the tile's scale) or exact (two words)")
    ap.add_argument("--weak", default=None, choices=["P-COLD", "P-WARM", "P-WEIBEL"],
                    help="weak scaling (SURVEY.md NEXT-2, PAPER.md:397-399): this config's grid per GPU, "
                         "the global grid grows along y with the GPU count")
    args = ap.parse_args()
    launch_ranks(args, sys.argv[1:])
    world, rank, local = dist_env()
    if args.weak:
        args.config = args.weak
    if args.impl == "reference":
        run_reference(args, world, rank)
        return

    numa_bind(local)
    import torch
    import synth
    import paper_2106_12485_b200 as z
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.weak:
        args.config = args.weak
    cfg = synth.config(args.config)
    if args.weak:   # fixed work per GPU: the slab of every rank is the config's grid
        cfg["ny"] *= world
        cfg["name"] += "-weak-%dgpu" % world
    if args.nx:
        cfg["nx"], cfg["ny"] = args.nx, args.ny or args.nx
        cfg["name"] += "-resized-%dx%d" % (cfg["nx"], cfg["ny"])
    dist_kw = None
    if world > 1:   # y-slabs, one per GPU, NCCL send/recv halos
        from paper_2106_12485_b200.dist import nccl_id_broadcast
        dist_kw = {"rank": rank, "world": world, "transport": args.transport, "nccl_id": nccl_id_broadcast(),
                   "device": local}
    sim = z.Simulation(cfg, inject=True, profile=not args.graphs, tile=args.tile, dist=dist_kw,
                       current_mode=args.current_mode, current_precision=args.current_precision)
    n_particles = sim.counters()["particles"]
    n_cells = cfg["nx"] * cfg["ny"]
    sim.step(args.warmup)
    sim.sync()
    sim.kernel_times()                 # reset the per-kernel accumulators
    launches0 = sim.counters()["launches"]
    clocks = ClockSampler(local)
    clocks.start()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(sim.torch_stream)
    step_ev = []
    if args.graphs:
        sim.step(args.steps)
    else:   # one event per step (the same launches): per-step statistics beside the total
        for _ in range(args.steps):
            sim.step(1)
            step_ev.append(torch.cuda.Event(enable_timing=True))
            step_ev[-1].record(sim.torch_stream)
    e1.record(sim.torch_stream)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    ms = e0.elapsed_time(e1)
    per_step, prev = [], e0
    for ev in step_ev:
        per_step.append(prev.elapsed_time(ev))
        prev = ev
    clk = clocks.stop()
    sim.sync()
    kt = sim.kernel_times()
    cnt = sim.counters()
    launches = cnt["launches"] - launches0
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
        npt = torch.tensor([n_particles], device="cuda", dtype=torch.int64)
        torch.distributed.all_reduce(npt)
        n_particles = int(npt.item())
    sim.close()

    k1_ms, k1_n = kt.get("k_push_tiles", (0.0, 0))
    k1_avg_s = k1_ms / max(k1_n, 1) * 1e-3 if k1_n else float("nan")
    k1_bytes = K1_BYTES_PER_PARTICLE * cnt["particles"] + K1_BYTES_PER_CELL * n_cells // max(world, 1)
    peak, peak_kind = measured_peaks()
    achieved = k1_bytes / k1_avg_s / 1e9 if k1_n else None
    traffic = k1_traffic(args.config, cfg["nx"], cfg["ny"]) if world == 1 else None
    value = n_particles * args.steps / (ms * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak" if args.weak else "strong",
        "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_name(args.config, cfg, n_particles),
                   "tile": cnt["tile"], "current_mode": ["reduction", "commutative"][args.current_mode],
                   "current_precision": args.current_precision,
                   "l2": "inputs larger than L2 (particle store %.1f GB)" % (n_particles * 24 / 1e9),
                   "parallelism": "y-slabs x%d" % world, "transport": args.transport if world > 1 else None},
        "cell_updates_per_s": n_cells * args.steps / (ms * 1e-3),
        "k1_pushes_per_s": cnt["particles"] / k1_avg_s if k1_n else None,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if k1_n else None,
                     "traffic": traffic,
                     # the same time against the ncu DRAM bytes, and the nominal 8 TB/s
                     "achieved_dram": traffic / k1_avg_s / 1e9 if (traffic and k1_n) else None,
                     "frac_dram": traffic / k1_avg_s / 1e9 / peak if (traffic and k1_n) else None,
                     "frac_nominal_8tbs": achieved / 8000.0 if k1_n else None,
                     "traffic_source": "profiles/r2_k1_traffic_c5.json (ncu dram__bytes_read+write, C5)",
                     "kernel": "k_push_tiles", "peak_kind": peak_kind,
                     "algorithmic_bytes_per_launch": k1_bytes, "avg_launch_ms": k1_avg_s * 1e3 if k1_n else None,
                     **({"note": "--graphs: CUDA-graph replay, no per-kernel events"} if args.graphs else {})},
        "kernel_ms_per_step": {k: v[0] / max(v[1], 1) for k, v in kt.items() if v[1]},
        # per-step times (CUDA events between the steps, this rank): the first / last steps show the
        # in-tile order decay
        **({"step_ms": {"mean": statistics.mean(per_step), "std": statistics.pstdev(per_step), "min": min(per_step),
                        "max": max(per_step), "first": per_step[0], "last": per_step[-1]}} if per_step else {}),
        "gpu_launches": launches,
        "cuda_graphs": bool(args.graphs),
        "clocks": clk,
    }
    if rank == 0 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(args)
    if not args.no_e2e:
        e2e = e2e_run(args, cfg, torch, z, dict(dist_kw, nccl_id=None) if dist_kw else None, world)
        if rank == 0:
            line["e2e"] = e2e
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
