"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same seeded
inputs (BASELINE.json north_star tolerances).  Needs a B200."""
import numpy as np
import pytest

import synth
from oracle.sim import from_config
from parity_util import (CELL_FRAC, CONT_TOL, ENERGY_TOL, FIELD_TOL, MOM_TOL, POS_TOL, compare_particles,
                         continuity_residual, energy_agreement, oracle_particles, rel_l2, rho_nodes)

pytestmark = pytest.mark.gpu


def _z():
    import paper_2106_12485_b200 as z
    return z


def gpu_from_particles(cfg, parts, tile=16, slack=1.25, current_mode=0):
    sim = _z().Simulation(cfg, inject=False, track_ids=True, tile=tile, capacity_slack=slack, current_mode=current_mode)
    for s, p in enumerate(parts):
        sim.set_particles(s, p)
    return sim


def _parity_run(cfg, steps, tile=16, check_every_step=True, slack=1.25, current_mode=0):
    parts = [synth.species_particles(cfg, s) for s in range(len(cfg["species"]))]
    g = gpu_from_particles(cfg, parts, tile, slack, current_mode)
    o = from_config(cfg, particles=parts)
    nx, ny, dx, dy, dt = cfg["nx"], cfg["ny"], cfg["dx"], cfg["dy"], cfg["dt"]
    per = (cfg["bc"][0] == 0, cfg["bc"][1] == 0)
    q = [o.species[s]["q"] for s in range(len(parts))]
    fe_g, fe_o, ke_g, ke_o = [], [], [], []
    prev = [g.particles(s, True) for s in range(len(parts))]
    prev_n = -1
    report = {}
    for n in range(steps):
        g.step(1)
        o.step()
        it, fe, ke = g.energy()
        assert it == n
        fe_g.append(fe); ke_g.append(ke)
        fe_o.append(o.fe[-1]); ke_o.append(o.ke[-1])
        if check_every_step or n in (0, 9, steps - 1):
            cur = [g.particles(s, True) for s in range(len(parts))]
            if n < 10 and prev_n == n - 1:
                rho0 = sum(rho_nodes(nx, ny, q[s], prev[s]) for s in range(len(parts)))
                rho1 = sum(rho_nodes(nx, ny, q[s], cur[s]) for s in range(len(parts)))
                r = continuity_residual(nx, ny, dx, dy, dt, rho0, rho1, g.fields(3), cfg["bc"])
                report.setdefault("continuity", []).append(r)
                assert r <= CONT_TOL, (n, r)
            if n == 0:
                for s in range(len(parts)):
                    c = compare_particles(cur[s], oracle_particles(o, s), nx, ny, per)
                    report["step1_s%d" % s] = c
                    assert c["pos_max"] <= POS_TOL, c
                    assert c["mom_max"] <= MOM_TOL, c
                    assert c["cell_exact_frac"] >= CELL_FRAC and c["cell_bad"] == 0, c
            if n == 9:
                eE, eB = rel_l2(g.fields(0), o.fields(0)), rel_l2(g.fields(1), o.fields(1))
                report["fields10"] = (eE, eB)
                assert eE <= FIELD_TOL and eB <= FIELD_TOL, (eE, eB)
                for s in range(len(parts)):
                    c = compare_particles(cur[s], oracle_particles(o, s), nx, ny, per)
                    assert c["cell_exact_frac"] >= CELL_FRAC, c
            prev, prev_n = cur, n
    assert energy_agreement(fe_g, fe_o) <= ENERGY_TOL
    for s in range(len(parts)):
        assert energy_agreement([k[s] for k in ke_g], [k[s] for k in ke_o]) <= ENERGY_TOL
    assert energy_agreement([f + sum(k) for f, k in zip(fe_g, ke_g)], [f + sum(k) for f, k in zip(fe_o, ke_o)]) <= ENERGY_TOL
    cnt = g.counters()
    assert cnt["particles"] == sum(len(s["ix"]) for s in o.species)
    g.close()
    return report


def test_c1_full_run():
    """BASELINE.json configs[0] at full size: 1-step particles, 10-step fields, 100-step energies."""
    cfg = synth.config("C1")
    rep = _parity_run(cfg, cfg["steps"], check_every_step=False)
    print(rep)


def test_c2_weibel_reduced():
    """configs[1] physics (two counter-streaming species) on a 64x64 grid, 12 steps."""
    cfg = synth.config("C2", nx=64, ny=64)
    _parity_run(cfg, 12)


@pytest.mark.parametrize("tile", [8, 16, 32])
def test_ragged_grid_tiles(tile):
    """Grid sizes that are not multiples of the tile (partial tiles on both axes)."""
    cfg = synth.config("C1", nx=50, ny=37)
    cfg["species"][0]["uth"] = (0.3, 0.3, 0.3)   # more crossings
    _parity_run(cfg, 10, tile=tile)


def test_c3_open_x_clouds_reduced():
    """configs[2] physics (two drifting clouds, open x: particles removed + Mur-1 fields,
    periodic y) on 128 x 32 cells, 40 steps (the clouds reach the open edges)."""
    cfg = synth.config("C3", nx=128, ny=32)
    cfg["species"][0].update(x0=0.0, x1=6.4)
    cfg["species"][1].update(x0=6.4, x1=12.8)
    rep = _parity_run(cfg, 40, check_every_step=False)
    print(rep)


def c4_reduced(nx=400, ny=64):
    """configs[3] physics on a smaller box: same dx, dy, dt, ppc, a0, omega0, fwhm, W0, filter and
    boundaries; the ramp starts at x = 2.0 (20 cells) and the laser's leading edge is Lx - 2."""
    cfg = synth.config("C4", nx=nx, ny=ny)
    cfg["species"][0].update(x0=2.0, x1=2.0 + 20 * cfg["dx"])
    cfg["laser"] = dict(cfg["laser"], start=nx * cfg["dx"] - 2.0)
    return cfg


def _gpu_c4(cfg, parts):
    g = gpu_from_particles(cfg, parts)
    E, B = synth.laser_fields(cfg)
    g.set_fields(0, E)
    g.set_fields(1, B)
    return g


def test_c4_lwfa_window_filter_reduced():
    """Moving window (shift + injection), compensated 4-pass filter, laser initial fields, density
    ramp and absorbing y edges, against the oracle: particles after 1 and 10 steps, fields after
    10 steps, energies over 30 steps (the window shifts on 28 of them)."""
    cfg = c4_reduced()
    parts = [synth.species_particles(cfg, 0)]
    g = _gpu_c4(cfg, parts)
    o = from_config(cfg, particles=parts)
    nx, ny = cfg["nx"], cfg["ny"]
    fe_g, fe_o, ke_g, ke_o = [], [], [], []
    for n in range(30):
        g.step(1)
        o.step()
        it, fe, ke = g.energy()
        fe_g.append(fe); ke_g.append(ke[0])
        fe_o.append(o.fe[-1]); ke_o.append(o.ke[-1][0])
        if n in (0, 9, 29):
            c = compare_particles(g.particles(0, True), oracle_particles(o, 0), nx, ny, (False, False))
            if n == 0:
                assert c["pos_max"] <= POS_TOL and c["mom_max"] <= MOM_TOL, c
            assert c["cell_exact_frac"] >= CELL_FRAC, c
        if n == 9:
            for w in (0, 1):
                assert rel_l2(g.fields(w), o.fields(w)) <= FIELD_TOL, (w, rel_l2(g.fields(w), o.fields(w)))
            # J and the charge density after 10 steps: measured 1.8e-7 and 1.7e-7 (round 2); the
            # bar is the fields' (north star 1e-4), tightened from round 1's 1e-3
            assert rel_l2(g.fields(3), o.fields(3)) <= FIELD_TOL
            assert rel_l2(g.fields(2), o.fields(2)) <= FIELD_TOL
    assert o.n_move == 28
    assert energy_agreement(fe_g, fe_o) <= ENERGY_TOL
    assert energy_agreement(ke_g, ke_o) <= ENERGY_TOL
    assert g.counters()["particles"] == len(o.species[0]["ix"])
    g.close()


@pytest.mark.parametrize("tile", [8, 16])
def test_paper_weibel_pairs_reduced(tile):
    """the paper's Weibel case, an electron and a positron
    cloud (m_q = -1, +1) counter-streaming along z at 256 ppc each, on 24 x 20 cells, 10 steps.
    16 x 16 tiles hold 2 x 65536 particles, 8 x 8 tiles 2 x 16384: both take the one-word current
    at S ~ 26 (a 4 x 4 window holds 8192 particles of charge 1/512: |J_node| <= 16)."""
    cfg = synth.config("P-WEIBEL", nx=24, ny=20)
    print(_parity_run(cfg, 10, tile=tile, check_every_step=False))


def test_paper_lwfa_16ppc_reduced():
    """the paper's LWFA case at 16 ppc: C4 physics (moving
    window, laser, ramp, compensated filter, absorbing y) on 300 x 48 cells, 12 steps."""
    cfg = synth.config("P-LWFA", nx=300, ny=48)
    cfg["species"][0].update(x0=2.0, x1=2.0 + 20 * cfg["dx"])
    cfg["laser"] = dict(cfg["laser"], start=cfg["nx"] * cfg["dx"] - 2.0)
    parts = [synth.species_particles(cfg, 0)]
    g = _gpu_c4(cfg, parts)
    o = from_config(cfg, particles=parts)
    fe_g, fe_o = [], []
    for n in range(12):
        g.step(1)
        o.step()
        fe_g.append(g.energy()[1])
        fe_o.append(o.fe[-1])
        if n == 0:
            c = compare_particles(g.particles(0, True), oracle_particles(o, 0), cfg["nx"], cfg["ny"], (False, False))
            assert c["pos_max"] <= POS_TOL and c["mom_max"] <= MOM_TOL and c["cell_exact_frac"] >= CELL_FRAC, c
        if n == 9:
            for w in (0, 1):
                assert rel_l2(g.fields(w), o.fields(w)) <= FIELD_TOL, (w, rel_l2(g.fields(w), o.fields(w)))
    assert o.n_move > 0
    assert energy_agreement(fe_g, fe_o) <= ENERGY_TOL
    assert g.counters()["particles"] == len(o.species[0]["ix"])
    g.close()


@pytest.mark.parametrize("name", ["C1", "C3"])
def test_commutative_current_mode(name):
    """SURVEY.md NEXT-4, the paper's "commutative" ghost-current variant:
    the tiles add their current blocks into J with global atomics instead of the K4 reduction;
    same parity bar (C1 full size 12 steps; C3 physics reduced, open x, 20 steps)."""
    if name == "C1":
        cfg = synth.config("C1")
    else:
        cfg = synth.config("C3", nx=128, ny=32)
        cfg["species"][0].update(x0=0.0, x1=6.4)
        cfg["species"][1].update(x0=6.4, x1=12.8)
    _parity_run(cfg, 12 if name == "C1" else 20, check_every_step=False, current_mode=1)


def test_cuda_graph_replay_matches_launches():
    """zpic_step(n) replays a captured two-step CUDA graph (single domain, no
    window); particles (keyed by id) and fields are bit-identical to plain launches (the tile
    current is an exact integer sum), for even and odd step counts."""
    cfg = synth.config("C1", nx=48, ny=40)
    cfg["species"][0]["uth"] = (0.3, 0.3, 0.3)
    parts = synth.species_particles(cfg, 0)
    out = []
    for graphs in (True, False):
        g = _z().Simulation(cfg, inject=False, track_ids=True, graphs=graphs)
        g.set_particles(0, parts)
        g.step(7)
        g.step(4)
        p = g.particles(0, True)
        o = np.argsort(p["id"])
        out.append(({k: v[o] for k, v in p.items()}, g.fields(0), g.fields(1), g.energy()))
        assert g.energy()[0] == 10
        g.close()
    (pa, Ea, Ba, ea), (pb, Eb, Bb, eb) = out
    for k in pa:
        assert np.array_equal(pa[k], pb[k]), k
    assert np.array_equal(Ea, Eb) and np.array_equal(Ba, Bb)
    # FE comes from the (identical) fields; KE is summed in fp32 per thread over the particles in
    # storage order, which K3's atomic insertion order leaves run-dependent: fp32-level agreement
    assert ea[1] == pytest.approx(eb[1], rel=1e-12) and ea[2][0] == pytest.approx(eb[2][0], rel=1e-6)


def test_window_injection_ids_and_counts():
    """Each shift injects ppc * ny particles per species at ix = nx - 1 with
    the oracle's ids; particles leaving x < 0 are removed."""
    cfg = c4_reduced(nx=160, ny=16)
    cfg["laser"] = dict(cfg["laser"], a0=0.0)
    parts = [synth.species_particles(cfg, 0)]
    g = _gpu_c4(cfg, parts)
    o = from_config(cfg, particles=parts)
    for n in range(12):
        g.step(1)
        o.step()
    gp = g.particles(0, True)
    assert len(gp["ix"]) == len(o.species[0]["ix"])
    assert np.array_equal(np.sort(gp["id"].astype(np.int64)), np.sort(o.species[0]["id"]))
    inj = gp["id"] >= 2 ** 31
    assert np.count_nonzero(inj) == o.n_move * 16 * 4
    g.close()


def test_mur_vacuum_matches_oracle():
    """Open x and open y edges with an initial random field and a pulse: the GPU's Mur-1
    boundary nodes follow the oracle (R13)."""
    for bc in ((1, 0), (0, 1), (1, 1), (2, 1), (2, 0)):
        cfg = synth.config("C1", nx=48, ny=40)
        cfg["bc"] = bc
        rng = np.random.default_rng(5)
        E = rng.normal(size=(3, 40, 48)).astype(np.float32)
        B = rng.normal(size=(3, 40, 48)).astype(np.float32)
        empty = {k: np.zeros(0, dt) for k, dt in (("ix", np.int32), ("iy", np.int32), ("x", np.float32),
                                                   ("y", np.float32), ("ux", np.float32), ("uy", np.float32),
                                                   ("uz", np.float32), ("id", np.uint32))}
        g = gpu_from_particles(cfg, [empty])
        g.set_fields(0, E)
        g.set_fields(1, B)
        o = from_config(cfg, particles=[empty], E=E, B=B)
        for _ in range(40):
            g.step(1)
            o.step()
        assert rel_l2(g.fields(0), o.fields(0)) < 1e-5, bc
        assert rel_l2(g.fields(1), o.fields(1)) < 1e-5, bc
        g.close()


def test_tile_overflow_loose_path():
    """Capacity slack 1.0: thermal fluctuations overflow tiles every step, so particles go
    through the loose list (global-memory push + re-insertion); results are unchanged."""
    cfg = synth.config("C1", nx=48, ny=48)
    cfg["species"][0]["uth"] = (0.4, 0.4, 0.4)
    _parity_run(cfg, 10, slack=1.0)


def test_hole_list_overflow_fallback():
    """A fast diagonal drift with 32x32 tiles makes > 256 particles leave a tile in one step,
    which exercises the sentinel compaction path of K1."""
    cfg = synth.config("C1", nx=64, ny=64)
    cfg["species"][0]["ufl"] = (2.0, 2.0, 0.0)
    cfg["species"][0]["uth"] = (0.05, 0.05, 0.05)
    _parity_run(cfg, 10, tile=32)


def test_device_injection_matches_generator():
    """K0 (device counter-based injector) reproduces synth's particles: positions bit-exact,
    momenta within 1 fp32 ulp (fp64 libm vs CUDA fp64 math)."""
    for name, over in (("C1", {}), ("C2", dict(nx=48, ny=40))):
        cfg = synth.config(name, **over)
        sim = _z().Simulation(cfg, inject=True, track_ids=True)
        for s in range(len(cfg["species"])):
            g = sim.particles(s, True)
            h = synth.species_particles(cfg, s)
            o = np.argsort(g["id"])
            g = {k: v[o] for k, v in g.items()}
            assert np.array_equal(g["id"], h["id"])
            for k in ("ix", "iy", "x", "y"):
                assert np.array_equal(g[k], h[k]), k
            for k in ("ux", "uy", "uz"):
                assert np.all(np.abs(g[k] - h[k]) <= np.spacing(np.abs(h[k]))), k
        sim.close()


def test_slab_injection_counts():
    cfg = synth.config("C3", nx=64, ny=32)
    cfg["species"][0].update(x0=0.0, x1=3.2)
    cfg["species"][1].update(x0=3.2, x1=6.4)
    cfg["bc"] = (0, 0)
    sim = _z().Simulation(cfg, inject=True, track_ids=True)
    for s in range(2):
        g = sim.particles(s, True)
        h = synth.species_particles(cfg, s)
        assert len(g["ix"]) == len(h["ix"]) == 32 * 32 * 8
        assert np.array_equal(np.sort(g["id"]), np.sort(h["id"]))
    sim.close()


def test_empty_and_vacuum():
    """No particles: fields stay exactly zero; a species with zero particles is allowed."""
    cfg = synth.config("C1", nx=32, ny=32)
    sim = _z().Simulation(cfg, inject=False, track_ids=True)
    sim.set_particles(0, {k: np.zeros(0, dt) for k, dt in
                          (("ix", np.int32), ("iy", np.int32), ("x", np.float32), ("y", np.float32),
                           ("ux", np.float32), ("uy", np.float32), ("uz", np.float32))})
    sim.step(5)
    for w in range(3):
        assert not np.any(sim.fields(w))
    assert sim.energy()[0] == 4
    sim.close()


def test_vacuum_wave_matches_oracle():
    """Pure field solve (K5 + guards): a random initial field, no particles, 50 steps."""
    cfg = synth.config("C1", nx=40, ny=24)
    rng = np.random.default_rng(3)
    E = rng.normal(size=(3, 24, 40)).astype(np.float32)
    B = rng.normal(size=(3, 24, 40)).astype(np.float32)
    empty = {k: np.zeros(0, dt) for k, dt in (("ix", np.int32), ("iy", np.int32), ("x", np.float32),
                                               ("y", np.float32), ("ux", np.float32), ("uy", np.float32),
                                               ("uz", np.float32), ("id", np.uint32))}
    g = gpu_from_particles(cfg, [empty])
    g.set_fields(0, E)
    g.set_fields(1, B)
    o = from_config(cfg, particles=[empty], E=E, B=B)
    for _ in range(50):
        g.step(1)
        o.step()
    assert rel_l2(g.fields(0), o.fields(0)) < 1e-5
    assert rel_l2(g.fields(1), o.fields(1)) < 1e-5
    g.close()


def _b_energy(sim, cfg):
    B = sim.fields(1).astype(np.float64)
    return 0.5 * cfg["dx"] * cfg["dy"] * float(np.sum(B * B))


def test_p12_weibel_field_growth_full_c2():
    """SURVEY.md P12 (physics sanity, not parity): in BASELINE.json's configs[1] (C2, full size,
    the 500-step run) the counter-streaming electrons filament and the magnetic energy grows by
    orders of magnitude (SPEC: B-energy(500) >= 10 x B-energy(10)); the total energy stays within
    a few per cent (leapfrog with a charge-conserving current)."""
    cfg = synth.config("C2")
    sim = _z().Simulation(cfg, inject=True)
    sim.step(10)
    b10 = _b_energy(sim, cfg)
    _, fe0, ke0 = sim.energy()
    sim.step(490)
    b500 = _b_energy(sim, cfg)
    it, fe, ke = sim.energy()
    assert it == 499
    assert b500 >= 10 * b10, (b10, b500)
    tot0, tot = fe0 + sum(ke0), fe + sum(ke)
    assert abs(tot - tot0) <= 0.05 * tot0, (tot0, tot)
    sim.close()


def test_p12_thermal_plasma_stable_full_c1():
    """P12: BASELINE.json configs[0] (C1, 100 steps): a uniform thermal plasma stays uniform and
    stable — kinetic energy drifts by < 2 %, the field energy stays a small fraction of it, and no
    particle is lost."""
    cfg = synth.config("C1")
    sim = _z().Simulation(cfg, inject=True)
    n0 = sim.counters()["particles"]
    sim.step(1)
    _, fe0, ke0 = sim.energy()
    sim.step(99)
    _, fe, ke = sim.energy()
    assert abs(ke[0] - ke0[0]) <= 0.02 * ke0[0], (ke0, ke)
    assert fe <= 0.05 * ke[0], (fe, ke)
    assert sim.counters()["particles"] == n0
    sim.close()


def test_repack_when_loose_list_grows():
    """Tile capacity slack 0.97: 3 % of the particles start in the loose list (global-memory
    push, re-inserted where slack appears) and thermal fluctuations keep it populated; at the
    check after 16 steps the library re-packs every species into tiles sized for the current
    largest tile (+10 %).  Same results as the oracle across the re-pack: the particle set (ids),
    fields after 18 steps, energies."""
    cfg = synth.config("C1", nx=128, ny=128)
    cfg["species"][0]["uth"] = (0.4, 0.4, 0.4)
    parts = [synth.species_particles(cfg, 0)]
    g = gpu_from_particles(cfg, parts, tile=16, slack=0.97)
    o = from_config(cfg, particles=parts)
    fe_g, fe_o = [], []
    for n in range(18):
        g.step(1)
        o.step()
        fe_g.append(g.energy()[1])
        fe_o.append(o.fe[-1])
    cnt = g.counters()
    assert cnt["repacks"] >= 1, cnt
    assert cnt["particles"] == len(parts[0]["ix"])
    c = compare_particles(g.particles(0, True), oracle_particles(o, 0), cfg["nx"], cfg["ny"])
    assert c["cell_exact_frac"] >= CELL_FRAC, c
    for w in (0, 1):
        assert rel_l2(g.fields(w), o.fields(w)) <= FIELD_TOL, (w, rel_l2(g.fields(w), o.fields(w)))
    assert energy_agreement(fe_g, fe_o) <= ENERGY_TOL
    g.close()


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_get_charge_diagnostic(name):
    """zpic_get_charge (SURVEY.md §8(b) diagnostics) equals the host-side bilinear node charge of
    the exported particles (R21), and with it the discrete continuity equation holds on the GPU
    path: |rho^{n+1} - rho^n + dt div J^{n+1/2}| <= 1e-5 (north star)."""
    cfg = synth.config(name, nx=48, ny=40)
    parts = [synth.species_particles(cfg, s) for s in range(len(cfg["species"]))]
    g = gpu_from_particles(cfg, parts)
    q = [synth.configs.charge(sp) for sp in cfg["species"]]
    rho0 = g.charge().astype(np.float64)
    host0 = sum(rho_nodes(cfg["nx"], cfg["ny"], q[s], g.particles(s)) for s in range(len(parts)))
    assert np.max(np.abs(rho0 - host0)) <= 1e-5 * max(1.0, np.max(np.abs(host0)))
    g.step(1)
    rho1 = g.charge().astype(np.float64)
    r = continuity_residual(cfg["nx"], cfg["ny"], cfg["dx"], cfg["dy"], cfg["dt"], rho0, rho1, g.fields(3), cfg["bc"])
    assert r <= CONT_TOL, r
    g.close()


@pytest.mark.parametrize("name", ["C4", "P-LWFA"])
def test_device_ramp_and_laser_match_generator(name):
    """zpic_init builds the density ramp (ZPIC_DENS_RAMP, R16) and the laser fields
    (zpic_options.laser, R17) on the device, in the library's own arithmetic; they agree with
    synth's generator: particles bit-exact (cold plasma: u = 0), E and B within 1 fp32 ulp."""
    cfg = synth.config(name, nx=300, ny=48)
    cfg["species"][0].update(x0=2.0, x1=2.0 + 20 * cfg["dx"])
    cfg["laser"] = dict(cfg["laser"], start=cfg["nx"] * cfg["dx"] - 2.0)
    sim = _z().Simulation(cfg, inject=True, track_ids=True)
    g = sim.particles(0, True)
    h = synth.species_particles(cfg, 0)
    o = np.argsort(g["id"])
    g = {k: v[o] for k, v in g.items()}
    assert np.array_equal(g["id"], h["id"])
    for k in ("ix", "iy", "x", "y", "ux", "uy", "uz"):
        assert np.array_equal(g[k], h[k]), k
    E, B = synth.laser_fields(cfg)
    for got, want in ((sim.fields(0), E), (sim.fields(1), B)):
        assert np.all(np.abs(got - want) <= np.spacing(np.abs(want)) + 1e-30)
    sim.close()


@pytest.mark.parametrize("shape", [(2, 2), (3, 5), (5, 3)])
def test_degenerate_tiny_grids(shape):
    """Grids smaller than a tile and than the 2-cell guard reach of the stencils (periodic images
    of a guard land on other guards or on the cell itself): same bars as C1 over 10 steps."""
    nx, ny = shape
    cfg = synth.config("C1", nx=nx, ny=ny)
    cfg["species"][0]["uth"] = (0.2, 0.2, 0.2)
    _parity_run(cfg, 10, check_every_step=False)


@pytest.mark.parametrize("shape", [(1, 4), (4, 1), (40000, 8)])
def test_invalid_grids_rejected(shape):
    """A grid one cell wide (a periodic image of the guard layer would be the cell itself twice)
    or beyond the 16-bit packed cell index is rejected at zpic_init with ZPIC_E_INVALID."""
    nx, ny = shape
    cfg = synth.config("C1", nx=nx, ny=ny)
    with pytest.raises(_z().ZpicError) as e:
        _z().Simulation(cfg, inject=True)
    assert e.value.status == -1


def test_cuda_graph_replay_moving_window():
    """With a moving window zpic_step replays one-step graphs keyed by (step parity, window
    shift) and the column injection reads the shift count from the device: particles (by id),
    fields and the injected ids match plain launches over 40 steps (38 shifts)."""
    out = []
    for graphs in (True, False):
        cfg = c4_reduced(nx=200, ny=32)
        sim = _z().Simulation(cfg, inject=True, track_ids=True, graphs=graphs)
        sim.step(40)
        p = sim.particles(0, True)
        o = np.argsort(p["id"])
        out.append(({k: v[o] for k, v in p.items()}, sim.fields(0), sim.fields(1)))
        sim.close()
    (pa, Ea, Ba), (pb, Eb, Bb) = out
    for k in pa:
        assert np.array_equal(pa[k], pb[k]), k
    assert np.array_equal(Ea, Eb) and np.array_equal(Ba, Bb)


def test_chunked_upload_validates_and_matches_direct_load():
    """zpic_set_particles streams a large upload (> 8 M particles) in chunks through two staging
    buffers into the tile store: the loaded set equals the input (keyed by id), and a particle with
    an offset outside [0, 1) anywhere in the upload is rejected with ZPIC_E_INVALID."""
    cfg = synth.config("C1", nx=768, ny=768)          # 9.4 M particles
    parts = synth.species_particles(cfg, 0)
    sim = _z().Simulation(cfg, inject=False, track_ids=True)
    sim.set_particles(0, parts)
    g = sim.particles(0, True)
    o = np.argsort(g["id"])
    g = {k: v[o] for k, v in g.items()}
    assert np.array_equal(g["id"], parts["id"])
    for k in ("ix", "iy", "x", "y", "ux", "uy", "uz"):
        assert np.array_equal(g[k], parts[k]), k
    bad = dict(parts)
    bad["x"] = parts["x"].copy()
    bad["x"][len(bad["x"]) - 3] = 1.0
    with pytest.raises(_z().ZpicError) as e:
        sim.set_particles(0, bad)
    assert e.value.status == -1
    sim.close()


@pytest.mark.parametrize("graphs,tile", [(False, 16), (True, 16), (False, 8)])
def test_periodic_resort_is_invisible(graphs, tile, monkeypatch):
    """K2s (the periodic in-tile re-sort) only permutes the slots of a tile: with a re-sort every
    step the fields (an exact integer current per tile) and every particle (by id) are
    bit-identical to a run without it, with and without CUDA-graph replay."""
    cfg = synth.config("C2", nx=72, ny=56)
    for sp in cfg["species"]:
        sp["uth"] = (0.3, 0.3, 0.3)
        sp["ppc"] = (2, 2)      # 16 x 16 tiles of 2 species x 1024 particles fit K2s's stage (7 words with ids)
    parts = [synth.species_particles(cfg, s) for s in range(2)]
    out = []
    sorted_tiles = []
    for every in ("1", "0"):
        monkeypatch.setenv("ZPIC_SORT_EVERY", every)
        g = _z().Simulation(cfg, inject=False, track_ids=True, tile=tile, capacity_slack=1.5, graphs=graphs)
        for s, p in enumerate(parts):
            g.set_particles(s, p)
        g.step(5)
        g.step(4)
        ps = []
        for s in range(2):
            p = g.particles(s, True)
            o = np.argsort(p["id"])
            ps.append({k: v[o] for k, v in p.items()})
        out.append((g.fields(0), g.fields(1), g.fields(2), ps, g.energy()))
        cnt = g.counters()
        sorted_tiles.append((cnt["sorted_tiles"], cnt["unsorted_tiles"]))
        g.close()
    assert sorted_tiles[0][0] > 0 and sorted_tiles[0][1] == 0, sorted_tiles    # K2s really ran on every tile
    assert sorted_tiles[1] == (0, 0)
    (Ea, Ba, Ja, pa, ea), (Eb, Bb, Jb, pb, eb) = out
    assert np.array_equal(Ja, Jb) and np.array_equal(Ea, Eb) and np.array_equal(Ba, Bb)
    for s in range(2):
        assert len(pa[s]["id"]) == len(parts[s]["x"])
        for k in pa[s]:
            assert np.array_equal(pa[s][k], pb[s][k]), (s, k)
    # KE is an fp32 sum in storage order: equal to fp32 accuracy
    assert ea[2][0] == pytest.approx(eb[2][0], rel=1e-6)


def test_resort_rank_overflow_and_crowded_cells(monkeypatch):
    """K2s with more particles in one cell than its key bitmap ranks (64 per cell at T = 16): the
    extra ranks go to the end of the tile in arbitrary order.  A cold cluster of 200 particles in
    one cell plus a thermal background; fields and particles (by id) bit-identical to no re-sort,
    and every particle survives."""
    cfg = synth.config("C1", nx=64, ny=64)
    cfg["species"][0]["uth"] = (0.2, 0.2, 0.2)
    cfg["species"][0]["ppc"] = (2, 2)     # 1024 per 16 x 16 tile (+ the cluster): fits K2s's stage
    bg = synth.species_particles(cfg, 0)
    rng = np.random.default_rng(7)
    k = 200
    cl = {"ix": np.full(k, 37, np.int32), "iy": np.full(k, 21, np.int32),
          "x": rng.random(k, dtype=np.float32), "y": rng.random(k, dtype=np.float32),
          "ux": np.zeros(k, np.float32), "uy": np.zeros(k, np.float32), "uz": np.zeros(k, np.float32),
          "id": (np.arange(k) + len(bg["x"])).astype(np.uint32)}
    parts = {f: np.concatenate([bg[f], cl[f]]) for f in bg}
    out = []
    for every in ("1", "0"):
        monkeypatch.setenv("ZPIC_SORT_EVERY", every)
        g = _z().Simulation(cfg, inject=False, track_ids=True, tile=16, capacity_slack=1.5)
        g.set_particles(0, parts)
        g.step(6)
        p = g.particles(0, True)
        o = np.argsort(p["id"])
        out.append(({f: v[o] for f, v in p.items()}, g.fields(0), g.fields(1)))
        if every == "1":
            cnt = g.counters()
            assert cnt["sorted_tiles"] > 0 and cnt["unsorted_tiles"] == 0, cnt
        g.close()
    (pa, Ea, Ba), (pb, Eb, Bb) = out
    assert len(pa["id"]) == len(parts["x"]) and np.array_equal(pa["id"], np.sort(parts["id"]))
    assert np.array_equal(Ea, Eb) and np.array_equal(Ba, Bb)
    for f in pa:
        assert np.array_equal(pa[f], pb[f]), f


def test_set_particles_replaces_the_species_loose_particles_included():
    """zpic_set_particles replaces a species: after steps that left particles in the loose list
    (tile slack 1.0), a new upload of that species is the whole species — nothing of the old set
    survives in the tiles or the loose list — and a rejected upload leaves it empty."""
    cfg = synth.config("C1", nx=48, ny=48)
    cfg["species"][0]["uth"] = (0.4, 0.4, 0.4)
    parts = synth.species_particles(cfg, 0)
    g = gpu_from_particles(cfg, [parts], slack=1.0)
    g.step(4)
    assert g.counters()["particles"] == len(parts["x"])
    half = {k: v[: len(v) // 2].copy() for k, v in parts.items()}
    g.set_particles(0, half)
    assert g.counters()["particles"] == len(half["x"])
    got = g.particles(0, True)
    assert np.array_equal(np.sort(got["id"]), np.sort(half["id"]))
    bad = dict(half)
    bad["x"] = half["x"].copy()
    bad["x"][3] = 1.5
    with pytest.raises(_z().ZpicError):
        g.set_particles(0, bad)
    assert g.counters()["particles"] == 0
    g.close()


@pytest.mark.parametrize("case", ["ragged8", "ragged32", "open_x", "window", "loose", "repack", "two_species"])
def test_occupancy_histogram_stays_exact(case, monkeypatch):
    """The per-tile cell histogram behind the fixed-point current's occupancy bound
    is maintained incrementally: K1 moves only its crossing particles, every insertion adds.  With
    ZPIC_CHECK_OCC=1 a recount before every step verifies it cell by cell, and that the bound covers
    the recount's largest 4 x 4 window (a violation stops the run with ZPIC_E_STATE), across partial
    tiles, open-edge removal, the moving window (shift + injection), the loose list, a re-pack and
    two species."""
    monkeypatch.setenv("ZPIC_CHECK_OCC", "1")
    slack, steps, tile = 1.25, 20, 16
    if case.startswith("ragged"):
        cfg = synth.config("C1", nx=50, ny=37)
        cfg["species"][0]["uth"] = (0.3, 0.3, 0.3)
        tile = int(case[6:])
    elif case == "open_x":
        cfg = synth.config("C3", nx=128, ny=32)
        cfg["species"][0].update(x0=0.0, x1=6.4)
        cfg["species"][1].update(x0=6.4, x1=12.8)
        steps = 40
    elif case == "window":
        cfg = c4_reduced(nx=200, ny=32)
        steps = 30
    elif case == "loose":
        cfg = synth.config("C1", nx=48, ny=48)
        cfg["species"][0]["uth"] = (0.4, 0.4, 0.4)
        slack = 1.0
    elif case == "repack":
        cfg = synth.config("C1", nx=128, ny=128)
        cfg["species"][0]["uth"] = (0.4, 0.4, 0.4)
        slack, steps = 0.97, 18
    else:
        cfg = synth.config("C2", nx=64, ny=64)
        for sp in cfg["species"]:
            sp["uth"] = (0.3, 0.3, 0.3)
    if case == "repack":   # an upload into tiles 3 % short of the lattice: loose list, re-pack at step 16
        g = gpu_from_particles(cfg, [synth.species_particles(cfg, 0)], tile=tile, slack=slack)
    else:
        g = _z().Simulation(cfg, inject=True, tile=tile, capacity_slack=slack)
    for _ in range(steps):
        g.step(1)
        g.counters()   # syncs and raises ZPIC_E_STATE on ERR_HIST
    if case == "repack":
        assert g.counters()["repacks"] >= 1
    if case == "loose":
        assert g.counters()["loose"] > 0 or g.counters()["repacks"] > 0
    g.close()


_FILTER_RUN = r"""
import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import synth, paper_2106_12485_b200 as z
nx, npass, comp, bcx, out = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
cfg = synth.config("C1", nx=nx, ny=48)
cfg["species"][0]["uth"] = (0.2, 0.2, 0.2)
cfg["filter"] = (npass, comp)
cfg["bc"] = (bcx, 0)
sim = z.Simulation(cfg, inject=True, tile=8, capacity_slack=2.0)
sim.step(8)
assert sim.counters()["loose"] == 0
np.savez(out, E=sim.fields(0), B=sim.fields(1), J=sim.fields(2))
"""


@pytest.mark.parametrize("nx,npass,comp,bcx", [(100, 4, 1, 0), (100, 4, 1, 1), (64, 1, 0, 0), (64, 7, 1, 1),
                                                (20, 2, 0, 1), (200, 4, 0, 0)])
def test_register_filter_is_bit_identical(tmp_path, nx, npass, comp, bcx):
    """The register form of the current filter (k_filter_x_reg: a window per thread, no shared
    memory) against the row-per-CTA form (ZPIC_FILTER_V1=1) over 8 steps of a plasma with the
    filter on: periodic and zero x guards, 1 to 8 passes, ragged and short rows (nx 20: every
    thread on the edge path).  The fixed-point current makes J independent of the particle order,
    so the two runs must agree bit for bit."""
    import os
    import subprocess
    import sys
    res = []
    for v1 in ("0", "1"):
        out = str(tmp_path / ("f%s.npz" % v1))
        env = dict(os.environ, ZPIC_FILTER_V1=v1)
        subprocess.check_call([sys.executable, "-c", _FILTER_RUN, str(nx), str(npass), str(comp), str(bcx), out],
                              env=env, cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        res.append(np.load(out))
    for k in ("E", "B", "J"):
        assert np.array_equal(res[0][k], res[1][k]), k
