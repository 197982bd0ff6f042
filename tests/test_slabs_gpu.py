"""y-slab decomposition on one B200 (P10 "regional deposit + ghost reduction
= global deposit", P virtual slabs = 1 slab).  Loopback groups step P slab contexts together
through the same exchange rounds the NCCL transport uses; the NCCL transport itself runs with a
one-rank self-ring.  Needs a B200."""
import numpy as np
import pytest

import synth
from oracle.sim import from_config
from parity_util import (CELL_FRAC, ENERGY_TOL, FIELD_TOL, MOM_TOL, POS_TOL, compare_particles, energy_agreement,
                         oracle_particles, rel_l2)

pytestmark = pytest.mark.gpu


def _z():
    import paper_2106_12485_b200 as z
    return z


def _group(cfg, world, parts, laser=False, **kw):
    from paper_2106_12485_b200.dist import LoopbackGroup
    g = LoopbackGroup(cfg, world, inject=False, track_ids=True, **kw)
    for s, p in enumerate(parts):
        g.set_particles(s, p)
    if laser:
        E, B = synth.laser_fields(cfg)
        g.set_fields(0, E)
        g.set_fields(1, B)
    return g


def _run_vs_oracle(cfg, world, steps, laser=False, **kw):
    parts = [synth.species_particles(cfg, s) for s in range(len(cfg["species"]))]
    g = _group(cfg, world, parts, laser, **kw)
    o = from_config(cfg, particles=parts)
    per = (cfg["bc"][0] == 0, cfg["bc"][1] == 0)
    fe_g, fe_o = [], []
    for n in range(steps):
        g.step(1)
        o.step()
        it, fe, ke = g.energy()
        assert it == n
        fe_g.append(fe + sum(ke))
        fe_o.append(o.fe[-1] + sum(o.ke[-1]))
        if n in (0, 9, steps - 1):
            for s in range(len(parts)):
                c = compare_particles(g.particles(s, True), oracle_particles(o, s), cfg["nx"], cfg["ny"], per)
                if n == 0:
                    assert c["pos_max"] <= POS_TOL and c["mom_max"] <= MOM_TOL, c
                assert c["cell_exact_frac"] >= CELL_FRAC, c
        if n == 9:
            for w in (0, 1):
                e = rel_l2(g.fields(w), o.fields(w))
                assert e <= FIELD_TOL, (w, e)
    assert energy_agreement(fe_g, fe_o) <= ENERGY_TOL
    assert g.counters()["particles"] == sum(len(s["ix"]) for s in o.species)
    g.close()


@pytest.mark.parametrize("world", [2, 4])
def test_slabs_periodic_c1(world):
    cfg = synth.config("C1", nx=48, ny=64)
    cfg["species"][0]["uth"] = (0.3, 0.3, 0.3)
    _run_vs_oracle(cfg, world, 12)


@pytest.mark.parametrize("world", [1, 2, 4])
def test_slabs_open_x_c3(world):
    cfg = synth.config("C3", nx=128, ny=32)
    cfg["species"][0].update(x0=0.0, x1=6.4, uth=(0.1, 0.1, 0.1))
    cfg["species"][1].update(x0=6.4, x1=12.8, uth=(0.1, 0.1, 0.1))
    _run_vs_oracle(cfg, world, 20)


@pytest.mark.parametrize("world", [2, 4])
def test_slabs_window_open_y_c4(world):
    cfg = synth.config("C4", nx=400, ny=64)
    cfg["species"][0].update(x0=2.0, x1=2.4)
    cfg["laser"] = dict(cfg["laser"], start=400 * cfg["dx"] - 2.0)
    _run_vs_oracle(cfg, world, 20, laser=True)


def test_slabs_equal_one_slab():
    """P = 4 virtual slabs reproduce the unsplit domain (P10) to fp32 summation order."""
    cfg = synth.config("C2", nx=64, ny=64)
    parts = [synth.species_particles(cfg, s) for s in range(2)]
    one = _z().Simulation(cfg, inject=False, track_ids=True)
    for s, p in enumerate(parts):
        one.set_particles(s, p)
    four = _group(cfg, 4, parts)
    for _ in range(15):
        one.step(1)
        four.step(1)
    for w in (0, 1, 2):
        assert rel_l2(four.fields(w), one.fields(w)) < 2e-5, w
    for s in range(2):
        c = compare_particles(four.particles(s, True), one.particles(s, True), 64, 64)
        assert c["pos_max"] < 1e-4 and c["cell_exact_frac"] >= CELL_FRAC, c
    one.close()
    four.close()


def test_nccl_transport_self_ring():
    """The NCCL transport (send / recv in groups on the compute stream) with one rank whose lower
    and upper neighbour is itself must reproduce the unsplit periodic domain."""
    z = _z()
    cfg = synth.config("C1", nx=48, ny=40)
    cfg["species"][0]["uth"] = (0.3, 0.3, 0.3)
    parts = [synth.species_particles(cfg, 0)]
    ref = z.Simulation(cfg, inject=False, track_ids=True)
    ref.set_particles(0, parts[0])
    uid = z.zpic.zpic_nccl_unique_id()
    ring = z.Simulation(cfg, inject=False, track_ids=True,
                        dist={"rank": 0, "world": 1, "transport": "nccl", "nccl_id": uid})
    ring.set_particles(0, parts[0])
    for _ in range(12):
        ref.step(1)
        ring.step(1)
    for w in (0, 1, 2):
        assert rel_l2(ring.fields(w), ref.fields(w)) < 2e-5, w
    c = compare_particles(ring.particles(0, True), ref.particles(0, True), 48, 40)
    assert c["pos_max"] < 1e-4 and c["cell_exact_frac"] >= CELL_FRAC, c
    assert abs(ring.energy()[1] - ref.energy()[1]) <= 1e-6 * max(abs(ref.energy()[1]), 1e-12)
    ring.close()
    ref.close()


@pytest.mark.parametrize("name", ["C1", "C3"])
def test_nccl_overlapped_rounds_self_ring(name):
    """The NCCL path overlaps round 1 (raw J rows + particles) with the Yee tile rows that need
    no halo and round 2 (E/B ghost rows) with the next step's K1 on interior tile rows, on a
    separate stream.  With a one-rank ring and 12 steps in one zpic_step call (every overlap in
    play: 10 K1 tile rows, 4 Yee tile rows), the result equals the unsplit domain."""
    z = _z()
    if name == "C1":
        cfg = synth.config("C1", nx=64, ny=160)
        cfg["species"][0]["uth"] = (0.3, 0.3, 0.3)
    else:
        cfg = synth.config("C3", nx=96, ny=160)
        cfg["species"][0].update(x0=0.0, x1=4.8)
        cfg["species"][1].update(x0=4.8, x1=9.6)
    parts = [synth.species_particles(cfg, s) for s in range(len(cfg["species"]))]
    ref = z.Simulation(cfg, inject=False, track_ids=True, graphs=False)
    uid = z.zpic.zpic_nccl_unique_id()
    ring = z.Simulation(cfg, inject=False, track_ids=True,
                        dist={"rank": 0, "world": 1, "transport": "nccl", "nccl_id": uid})
    for s, p in enumerate(parts):
        ref.set_particles(s, p)
        ring.set_particles(s, p)
    ref.step(12)
    ring.step(12)
    for w in (0, 1, 2):
        assert rel_l2(ring.fields(w), ref.fields(w)) < 2e-5, w
    for s in range(len(parts)):
        c = compare_particles(ring.particles(s, True), ref.particles(s, True), cfg["nx"], cfg["ny"],
                              (cfg["bc"][0] == 0, True))
        assert c["pos_max"] < 1e-4 and c["cell_exact_frac"] >= CELL_FRAC, c
    assert abs(ring.energy()[1] - ref.energy()[1]) <= 1e-6 * max(abs(ref.energy()[1]), 1e-12)
    ring.close()
    ref.close()


@pytest.mark.parametrize("name", ["C1", "C3"])
def test_nccl_slab_graph_replay_matches_launches(name):
    """SURVEY.md NEXT-1 on the slab path: zpic_step(n) on the NCCL transport replays two-step CUDA
    graphs (both halo rounds captured with the comm-stream fork / join and their overlap with the
    interior kernels).  With a one-rank ring, 11 steps (five graph replays + one plain step) give
    the same fields and particles (by id) as plain launches, bit for bit (the tile current is an
    exact integer sum; no loose particles at this slack)."""
    z = _z()
    if name == "C1":
        cfg = synth.config("C1", nx=64, ny=96)
        cfg["species"][0]["uth"] = (0.3, 0.3, 0.3)
    else:
        cfg = synth.config("C3", nx=96, ny=96)
        cfg["species"][0].update(x0=0.0, x1=4.8)
        cfg["species"][1].update(x0=4.8, x1=9.6)
    parts = [synth.species_particles(cfg, s) for s in range(len(cfg["species"]))]
    out = []
    for graphs in (True, False):
        uid = z.zpic.zpic_nccl_unique_id()
        ring = z.Simulation(cfg, inject=False, track_ids=True, graphs=graphs, capacity_slack=1.5,
                            dist={"rank": 0, "world": 1, "transport": "nccl", "nccl_id": uid})
        for s, p in enumerate(parts):
            ring.set_particles(s, p)
        ring.step(7)
        ring.step(4)
        ps = []
        for s in range(len(parts)):
            p = ring.particles(s, True)
            o = np.argsort(p["id"])
            ps.append({k: v[o] for k, v in p.items()})
        out.append((ring.fields(0), ring.fields(1), ps, ring.energy()[0]))
        ring.close()
    (Ea, Ba, pa, ia), (Eb, Bb, pb, ib) = out
    assert ia == ib == 10
    assert np.array_equal(Ea, Eb) and np.array_equal(Ba, Bb)
    for s in range(len(parts)):
        for k in pa[s]:
            assert np.array_equal(pa[s][k], pb[s][k]), (s, k)


PEER_CASES = [(n, w, cm) for n in ("C1", "C3", "C4") for w in (2, 4) for cm in (0, 1)]


@pytest.mark.parametrize("name,world,current_mode", PEER_CASES)
def test_loopback_peer_transport_matches_oracle(name, world, current_mode):
    """The PEER transport's kernels in a loopback group against the oracle (particles after 1,
    10 and the last step, fields after 10, energies): current_mode 0 = the reduction (raw J rows
    and particles written into the neighbours' receive areas, epoch flags), 1 = the cross-slab
    "commutative" current (the slab-edge tiles and loose particles add their
    ghost rows straight into the neighbours' J; "zeroed" flags before any K1, the x-guard fold
    after the round-1 wait).  C1 periodic, C3 open x, C4 window + filter + open y."""
    if name == "C1":
        cfg = synth.config("C1", nx=48, ny=64)
        cfg["species"][0]["uth"] = (0.3, 0.3, 0.3)
        _run_vs_oracle(cfg, world, 12, transport="loopback_peer", current_mode=current_mode)
    elif name == "C3":
        cfg = synth.config("C3", nx=128, ny=32)
        cfg["species"][0].update(x0=0.0, x1=6.4, uth=(0.1, 0.1, 0.1))
        cfg["species"][1].update(x0=6.4, x1=12.8, uth=(0.1, 0.1, 0.1))
        _run_vs_oracle(cfg, world, 20, transport="loopback_peer", current_mode=current_mode)
    else:
        cfg = synth.config("C4", nx=400, ny=64)
        cfg["species"][0].update(x0=2.0, x1=2.4)
        cfg["laser"] = dict(cfg["laser"], start=400 * cfg["dx"] - 2.0)
        _run_vs_oracle(cfg, world, 20, laser=True, transport="loopback_peer", current_mode=current_mode)


@pytest.mark.parametrize("name", ["C1", "C3", "C4"])
def test_loopback_peer_equals_loopback_copies(name):
    """PEER rounds vs the device-copy rounds of the same loopback group (periodic y, open x, and
    C4's window + open y chain): the same particles (by id) and fields, bit for bit."""
    if name == "C1":
        cfg = synth.config("C1", nx=48, ny=64)
        cfg["species"][0]["uth"] = (0.3, 0.3, 0.3)
    elif name == "C3":
        cfg = synth.config("C3", nx=96, ny=64)
        cfg["species"][0].update(x0=0.0, x1=4.8)
        cfg["species"][1].update(x0=4.8, x1=9.6)
    else:
        cfg = synth.config("C4", nx=200, ny=32)
        cfg["species"][0].update(x0=2.0, x1=2.0 + 20 * cfg["dx"])
        cfg["laser"] = dict(cfg["laser"], start=cfg["nx"] * cfg["dx"] - 2.0)
    parts = [synth.species_particles(cfg, s) for s in range(len(cfg["species"]))]
    from paper_2106_12485_b200.dist import LoopbackGroup
    out = []
    for tr in ("loopback", "loopback_peer"):
        g = LoopbackGroup(cfg, 4, transport=tr, inject=False, track_ids=True, capacity_slack=1.5)
        for s, p in enumerate(parts):
            g.set_particles(s, p)
        if name == "C4":
            E, B = synth.laser_fields(cfg)
            g.set_fields(0, E)
            g.set_fields(1, B)
        g.step(10)
        ps = []
        for s in range(len(parts)):
            p = g.particles(s, True)
            o = np.argsort(p["id"])
            ps.append({k: v[o] for k, v in p.items()})
        out.append((g.fields(0), g.fields(1), ps))
        g.close()
    (Ea, Ba, pa), (Eb, Bb, pb) = out
    assert np.array_equal(Ea, Eb) and np.array_equal(Ba, Bb)
    for s in range(len(parts)):
        for k in pa[s]:
            assert np.array_equal(pa[s][k], pb[s][k]), (s, k)


@pytest.mark.parametrize("name,current_mode", [("C1", 0), ("C3", 0), ("C1", 1), ("C3", 1)])
def test_peer_transport_self_ring(name, current_mode):
    """ZPIC_TRANSPORT_PEER with one rank: the ring's neighbour is the context itself, so every
    round goes through the put / signal / wait kernels on its own receive block (round 2 pending
    into the next step's boundary K1, as across GPUs); with current_mode 1 the slab-edge tiles add
    their ghost rows into their own J through the peer path (the periodic y fold).  Equal to the
    unsplit domain."""
    z = _z()
    if name == "C1":
        cfg = synth.config("C1", nx=64, ny=160)
        cfg["species"][0]["uth"] = (0.3, 0.3, 0.3)
    else:
        cfg = synth.config("C3", nx=96, ny=160)
        cfg["species"][0].update(x0=0.0, x1=4.8)
        cfg["species"][1].update(x0=4.8, x1=9.6)
    parts = [synth.species_particles(cfg, s) for s in range(len(cfg["species"]))]
    ref = z.Simulation(cfg, inject=False, track_ids=True, graphs=False, current_mode=current_mode)
    ring = z.Simulation(cfg, inject=False, track_ids=True, dist={"rank": 0, "world": 1, "transport": "peer"},
                        current_mode=current_mode)
    for s, p in enumerate(parts):
        ref.set_particles(s, p)
        ring.set_particles(s, p)
    ref.step(12)
    ring.step(7)
    ring.step(5)
    for w in (0, 1, 2):
        assert rel_l2(ring.fields(w), ref.fields(w)) < 2e-5, w
    for s in range(len(parts)):
        c = compare_particles(ring.particles(s, True), ref.particles(s, True), cfg["nx"], cfg["ny"],
                              (cfg["bc"][0] == 0, True))
        assert c["pos_max"] < 1e-4 and c["cell_exact_frac"] >= CELL_FRAC, c
    ring.close()
    ref.close()


@pytest.mark.parametrize("commutative", [False, True])
@pytest.mark.parametrize("ranks,periodic", [(1, True), (2, True), (3, True), (8, True), (4, False), (17, True)])
def test_peer_protocol_under_concurrency(ranks, periodic, commutative):
    """The PEER halo protocol with the transport's own put / signal / wait code, every emulated
    slab a CTA of one cooperative launch (zpic_peer_selftest): 300 steps of both rounds with waits
    that really spin on flags other CTAs store concurrently (the loopback groups never spin), every
    received value checked against what its sender wrote for that step; with the cross-slab
    commutative current the shared J rows must hold exactly the own plus the neighbour's adds."""
    z = _z()
    bad, timeouts = z.zpic.zpic_peer_selftest(ranks, 300, 200, 16, 256, periodic, commutative)
    assert (bad, timeouts) == (0, 0)


def test_peer_protocol_selftest_detects_faults():
    """The self-test is not vacuous: a value corrupted in flight is counted, and a signal that never
    comes ends the neighbours' waits at the cycle budget instead of hanging."""
    z = _z()
    for cm in (False, True):
        bad, timeouts = z.zpic.zpic_peer_selftest(4, 10, 200, 16, 256, True, cm, fault=1)
        assert bad >= 1 and timeouts == 0
        bad, timeouts = z.zpic.zpic_peer_selftest(4, 10, 200, 16, 256, True, cm, budget_cycles=200_000_000, fault=2)
        assert timeouts >= 2
