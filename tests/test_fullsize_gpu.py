"""Parity at BASELINE.json's full sizes (north-star tolerances).  C2 and C4 are small enough for
the oracle to run whole; C3 runs the oracle for 10 steps on the full grid; C5 (1.07e9 particles,
in the launch configuration bench.py times: device injector, 16x16 tiles) is checked on sampled
patches: the oracle re-runs a periodic patch of the global lattice (rebuilt from the seeded
generator with global ids) and, since fields and particles travel at most one cell per step, the
patch interior beyond a margin of k+2 cells is exact after k steps.  Needs a B200."""
import numpy as np
import pytest

import synth
from oracle.sim import OracleSim, from_config
from parity_util import (CELL_FRAC, ENERGY_TOL, FIELD_TOL, MOM_TOL, POS_TOL, compare_particles, energy_agreement,
                         oracle_particles, rel_l2)

pytestmark = pytest.mark.gpu


def _z():
    import paper_2106_12485_b200 as z
    return z


def _full_run(cfg, steps, laser=False, check_cells=True):
    parts = [synth.species_particles(cfg, s) for s in range(len(cfg["species"]))]
    g = _z().Simulation(cfg, inject=False, track_ids=True)
    for s, p in enumerate(parts):
        g.set_particles(s, p)
    E = B = None
    if laser:
        E, B = synth.laser_fields(cfg)
        g.set_fields(0, E)
        g.set_fields(1, B)
    o = from_config(cfg, particles=parts, E=E, B=B)
    per = (cfg["bc"][0] == 0, cfg["bc"][1] == 0)
    tot_g, tot_o = [], []
    for n in range(steps):
        g.step(1)
        o.step()
        _, fe, ke = g.energy()
        tot_g.append(fe + sum(ke))
        tot_o.append(o.fe[-1] + sum(o.ke[-1]))
        if n in (0, steps - 1):
            for s in range(len(parts)):
                c = compare_particles(g.particles(s, True), oracle_particles(o, s), cfg["nx"], cfg["ny"], per)
                if n == 0:
                    assert c["pos_max"] <= POS_TOL and c["mom_max"] <= MOM_TOL, c
                if check_cells:
                    assert c["cell_exact_frac"] >= CELL_FRAC, c
        if n == 9:
            for w in (0, 1):
                e = rel_l2(g.fields(w), o.fields(w))
                assert e <= FIELD_TOL, (w, e)
    assert energy_agreement(tot_g, tot_o) <= ENERGY_TOL
    g.close()


def test_c2_full_size():
    cfg = synth.config("C2")          # 256^2, 2 x 1,048,576 particles
    _full_run(cfg, 12)


def test_c3_full_size():
    cfg = synth.config("C3")          # 2048 x 1024, 16.8 M particles, open x
    _full_run(cfg, 10)


def test_c4_full_size():
    cfg = synth.config("C4")          # 4000 x 512, 6.1 M particles, window, filter, laser
    _full_run(cfg, 10, laser=True)


def test_c5_full_size_sampled_patches():
    z = _z()
    cfg = synth.config("C5")
    k, W, m = 3, 64, 5
    sim = z.Simulation(cfg, inject=True, tile=16)       # bench.py's launch configuration
    assert sim.counters()["particles"] == 8192 * 8192 * 16
    sim.step(k)
    F = [sim.fields(w) for w in (0, 1, 2)]
    cnt = sim.counters()
    assert cnt["particles"] == 8192 * 8192 * 16
    sim.close()
    for gx0, gy0 in ((1000, 3000), (8192 - 30, 8192 - 20), (4090, 6140)):   # interior, both seams, tile edges
        p = synth.generate.patch_species(cfg, 0, gx0, gy0, W, W)
        sp = dict(cfg["species"][0])
        sp.update(p)
        o = OracleSim(W, W, cfg["dx"], cfg["dy"], cfg["dt"], [sp])
        o.run(k)
        ys = (gy0 + np.arange(W)) % 8192
        xs = (gx0 + np.arange(W)) % 8192
        for w in (0, 1, 2):
            got = F[w][:, ys][:, :, xs][:, m:W - m, m:W - m]
            want = o.fields(w)[:, m:W - m, m:W - m]
            e = rel_l2(got, want)
            assert e <= FIELD_TOL, (gx0, gy0, w, e)
