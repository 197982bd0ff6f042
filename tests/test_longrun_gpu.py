"""Every BASELINE.json workload for its full step count on the GPU (C1 100, C2 500, C3 1000, C4
4000, C5 50 steps): the run completes without a capacity or migration error (tile slack, the
mailboxes, the loose list and the re-pack path absorb the density changes of filamentation,
colliding clouds and the wakefield), particles are conserved where the boundaries conserve them,
and the total energy stays bounded.  Needs a B200."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


def _z():
    import paper_2106_12485_b200 as z
    return z


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_full_length_run(name):
    cfg = synth.config(name)
    sim = _z().Simulation(cfg, inject=True)   # device init: lattices, C4's ramp and laser
    n0 = sim.counters()["particles"]
    sim.step(1)
    _, fe0, ke0 = sim.energy()
    tot0 = fe0 + sum(ke0)
    sim.step(cfg["steps"] - 1)
    it, fe, ke = sim.energy()
    cnt = sim.counters()
    print(name, "steps", it + 1, "particles", n0, "->", cnt["particles"], "repacks", cnt["repacks"],
          "energy", tot0, "->", fe + sum(ke))
    assert it == cfg["steps"] - 1
    if cfg["bc"] == (0, 0):
        assert cnt["particles"] == n0
    assert np.isfinite(fe) and all(np.isfinite(k) for k in ke)
    if name in ("C1", "C2", "C5"):   # periodic, no injection: the energy is conserved to a few %
        assert abs(fe + sum(ke) - tot0) <= 0.05 * tot0, (tot0, fe + sum(ke))
    sim.close()


def test_full_length_c2_with_periodic_resort(monkeypatch):
    """C2 (Weibel filamentation, 500 steps) with a K2s re-sort every 16 steps against the same run
    without it.  The re-sort only permutes slots and the tile current is an exact integer sum, so
    with tile slack large enough that no particle ever goes loose (loose particles add into J with
    fp32 atomics, whose order varies between runs) the two runs are bit-identical; every tile was
    sorted (its particles fit the re-sort stage) and no particle went loose."""
    cfg = synth.config("C2")
    for sp in cfg["species"]:
        sp["ppc"] = (2, 2)     # 8 x 8 tiles: 2 x 256 particles per tile, slack 8 absorbs the filaments
    out = []
    for every in ("0", "16"):
        monkeypatch.setenv("ZPIC_SORT_EVERY", every)
        sim = _z().Simulation(cfg, inject=True, tile=8, capacity_slack=8.0)
        loose = 0
        for _ in range(cfg["steps"] // 50):
            sim.step(50)
            loose = max(loose, sim.counters()["loose"])
        assert loose == 0, loose      # no particle ever went loose: the run is bit-reproducible
        cnt = sim.counters()
        out.append((sim.fields(0), sim.fields(1), cnt))
        sim.close()
    (E0, B0, c0), (Es, Bs, cs) = out
    assert c0["particles"] == cs["particles"] == 256 * 256 * 8
    assert c0["repacks"] == 0 and cs["repacks"] == 0, (c0, cs)
    assert cs["sorted_tiles"] > 0 and cs["unsorted_tiles"] == 0, cs
    assert np.array_equal(E0, Es) and np.array_equal(B0, Bs)
