"""Full-length parity against the fp64 oracle (BASELINE.json north_star; SURVEY.md §8(c)
R19-R23): every BASELINE config at full size — C1 and C2 for their whole runs (100, 500 steps),
C3 and C4 for 200 steps, C5 (1.07e9 particles, the launch configuration bench.py times) on
sampled patches for its whole 50-step run.  Checked: the discrete continuity residual of the GPU's
own charge and pre-filter current (R21, <= 1e-5) every step (C1, C2) or every 10th step (C3, C4),
the FE / KE_s / total energy histories (R22, within 1 %), E and B after 10 steps (R20, <= 1e-4),
the particle count, and the final field maps the way PAPER.md:351-353 validates (relative error
of the last B map; the paper reports ~1e-4 between its fp32 variants).  The oracle runs start in
background processes when this module is collected (tests/conftest.py), so they overlap the rest
of the GPU suite.  Needs a B200."""
import json
import os

import numpy as np
import pytest

import fullrun_specs as F
import synth
from parity_util import CONT_TOL, ENERGY_TOL, FIELD_TOL, continuity_residual, energy_agreement, rel_l2

pytestmark = pytest.mark.gpu

# Final-map bars (reading): fp32 roundoff grows over a long run; the paper's own
# fp32 implementations differ by ~1e-4 in the final B map.  Here the final B map
# must stay within 1e-3 relative L2 of the fp64 oracle (measured: C2 after 500 Weibel steps 1.2e-4,
# C1-C5 <= 8e-5) and E within 1e-2 (E is ~100x weaker than B in the Weibel run: 8e-4 measured).
FINAL_B_TOL = 1e-3
FINAL_E_TOL = 1e-2


def _z():
    import paper_2106_12485_b200 as z
    return z


def _report(name, rec):
    d = os.environ.get("ZPIC_REPORT_DIR")
    print(name, json.dumps(rec))
    if d:
        os.makedirs(d, exist_ok=True)
        with open(os.path.join(d, "fullrun_%s.json" % name), "w") as f:
            json.dump(rec, f, indent=1)


def _max_rel(a, b):
    return float(np.max(np.abs(a.astype(np.float64) - b)) / max(np.max(np.abs(b)), 1e-30))


def _gpu_run(name, precision, cont_every):
    cfg, parts, E, B = F.inputs(name)
    _, steps, snaps = F.RUNS[name]
    g = _z().Simulation(cfg, inject=False, current_precision=precision)
    for s, p in enumerate(parts):
        g.set_particles(s, p)
    if E is not None:
        g.set_fields(0, E)
        g.set_fields(1, B)
    nx, ny, dx, dy, dt = cfg["nx"], cfg["ny"], cfg["dx"], cfg["dy"], cfg["dt"]
    checked = {n for n in range(steps) if (n + 1) % cont_every == 0 or n < 3 or n == steps - 1}
    fe, ke, cont, fields = [], [], [], {}
    n_move = 0
    rho_prev = None   # the charge after the previous step, when it was taken
    for n in range(steps):
        rho0 = (rho_prev if rho_prev is not None else g.charge().astype(np.float64)) if n in checked else None
        g.step(1)
        it, f, k = g.energy()
        assert it == n
        fe.append(f)
        ke.append(k)
        shifted = cfg["bc"][0] == 2 and (n + 1) * dt > dx * (n_move + 1)
        n_move += shifted
        rho_prev = None
        if n in checked:
            rho1 = g.charge().astype(np.float64)
            # R21: rho from the positions after the push, before the window shift (undone here)
            r1 = np.roll(rho1, 1, axis=1) if shifted else rho1
            cont.append((n, continuity_residual(nx, ny, dx, dy, dt, rho0, r1, g.fields(3), cfg["bc"])))
            rho_prev = rho1
        if n + 1 in snaps:
            fields[n + 1] = (g.fields(0), g.fields(1))
    cnt = g.counters()
    g.close()
    return cfg, np.array(fe), np.array(ke), cont, fields, cnt


# C3 and C4 for their whole 1000 / 4000 steps: the oracle needs ~27 / ~46 minutes, so these run
# only with ZPIC_FULLRUN_LONG=1 (reports: profiles/r2_fullrun_whole/)
_LONG = [pytest.param("C3-whole", "auto", 50, marks=pytest.mark.oracle_run("C3-whole")),
         pytest.param("C4-whole", "auto", 100, marks=pytest.mark.oracle_run("C4-whole"))] \
    if os.environ.get("ZPIC_FULLRUN_LONG") == "1" else []


@pytest.mark.parametrize("name,precision,cont_every", [
    pytest.param("C1", "auto", 1, marks=pytest.mark.oracle_run("C1")),
    pytest.param("C2", "auto", 1, marks=pytest.mark.oracle_run("C2")),
    pytest.param("C2", "exact", 1, marks=pytest.mark.oracle_run("C2")),
    pytest.param("C3", "auto", 10, marks=pytest.mark.oracle_run("C3")),
    pytest.param("C4", "auto", 10, marks=pytest.mark.oracle_run("C4")),
] + _LONG)
def test_full_run_parity(name, precision, cont_every, oracle_run):
    cfg, fe, ke, cont, fields, cnt = _gpu_run(name, precision, cont_every)
    o = oracle_run(name)
    _, steps, snaps = F.RUNS[name]
    rec = {"config": name, "steps": steps, "current_precision": precision, "oracle_seconds": float(o["seconds"])}
    # R21 continuity, every checked step
    rec["continuity_max"] = max(r for _, r in cont)
    rec["continuity_checked_steps"] = len(cont)
    rec["continuity"] = cont
    # R22 energy histories
    rec["fe_agreement"] = energy_agreement(fe, o["fe"])
    rec["ke_agreement"] = [energy_agreement(ke[:, s], o["ke"][:, s]) for s in range(ke.shape[1])]
    rec["total_agreement"] = energy_agreement(fe + ke.sum(1), o["fe"] + o["ke"].sum(1))
    # R20 after 10 steps, and the final maps
    E10, B10 = fields[10]
    rec["E10_rel_l2"], rec["B10_rel_l2"] = rel_l2(E10, o["E10"]), rel_l2(B10, o["B10"])
    Ef, Bf = fields[steps]
    rec["E_final_rel_l2"], rec["B_final_rel_l2"] = rel_l2(Ef, o["E%d" % steps]), rel_l2(Bf, o["B%d" % steps])
    rec["B_final_max_rel"] = _max_rel(Bf, o["B%d" % steps])
    rec["particles"] = [int(cnt["particles"]), int(o["particles"].sum())]
    whole = name.endswith("-whole")
    if whole:
        # the whole unstable runs: the same GPU run with the exact two-word current differs from this
        # one only in rounding; its distance is the run's own predictability limit (the counter-
        # streaming clouds amplify any rounding difference, tools/gpu/divergence.py)
        _, _, _, fields_x, _ = _gpu_run(name, "exact", 10 ** 9)[1:]
        Ex, Bx = fields_x[steps]
        rec["E_final_gpu_vs_gpu"], rec["B_final_gpu_vs_gpu"] = rel_l2(Ef, Ex), rel_l2(Bf, Bx)
    _report("%s_%s" % (name, precision), rec)
    assert rec["continuity_max"] <= CONT_TOL, rec
    assert rec["fe_agreement"] <= ENERGY_TOL and max(rec["ke_agreement"]) <= ENERGY_TOL, rec
    assert rec["total_agreement"] <= ENERGY_TOL, rec
    assert rec["E10_rel_l2"] <= FIELD_TOL and rec["B10_rel_l2"] <= FIELD_TOL, rec
    if whole:
        # PAPER.md:351-353 compares final maps of implementations that differ only in rounding
        # (~1e-4 there); past the instability's saturation the GPU-vs-oracle distance must stay
        # within 3x the GPU's own rounding-only divergence, and the particle count (open edges)
        # within 1e-5
        assert rec["B_final_rel_l2"] <= 3 * rec["B_final_gpu_vs_gpu"] + FINAL_B_TOL, rec
        assert rec["E_final_rel_l2"] <= 3 * rec["E_final_gpu_vs_gpu"] + FINAL_E_TOL, rec
        assert abs(rec["particles"][0] - rec["particles"][1]) <= 1e-5 * rec["particles"][1], rec
    else:
        assert rec["B_final_rel_l2"] <= FINAL_B_TOL and rec["E_final_rel_l2"] <= FINAL_E_TOL, rec
        assert rec["particles"][0] == rec["particles"][1], rec


@pytest.mark.oracle_run("C5")
@pytest.mark.parametrize("precision", ["auto", "exact"])
def test_c5_full_run_sampled_patches(precision, oracle_run):
    """C5 in bench.py's launch configuration (device injector, 16 x 16 tiles) for its whole
    50-step run: the fields of three patch interiors (margin 2k + 4 cells) at steps 1, 10, 25, 50
    against the oracle run on the periodic patch of the global lattice (R20 at step 10, the
    patch-interior field energy within 1 %, the final map within the final-map bar), and the
    discrete continuity of the full 8192^2 grid (R21) after steps 1, 2 and 50."""
    z = _z()
    cfg = synth.config("C5")
    nx, ny, dx, dy, dt = cfg["nx"], cfg["ny"], cfg["dx"], cfg["dy"], cfg["dt"]
    sim = z.Simulation(cfg, inject=True, tile=16, current_precision=precision)
    n0 = sim.counters()["particles"]
    assert n0 == nx * ny * 16
    W, m = F.C5_PATCH, F.C5_MARGIN
    got = {}
    cont = []
    rho0 = sim.charge().astype(np.float64)
    for n in range(1, F.C5_STEPS + 1):
        sim.step(1)
        if n in (1, 2, F.C5_STEPS):
            rho1 = sim.charge().astype(np.float64)
            cont.append((n, continuity_residual(nx, ny, dx, dy, dt, rho0, rho1, sim.fields(3), cfg["bc"])))
        if n in (1, F.C5_STEPS - 1):
            rho0 = sim.charge().astype(np.float64)
        if n in F.C5_SNAPS:
            E, B = sim.fields(0), sim.fields(1)
            for k, (gx0, gy0) in enumerate(F.C5_ORIGINS):
                ys = (gy0 + np.arange(W)) % ny
                xs = (gx0 + np.arange(W)) % nx
                got[(k, n)] = (E[:, ys][:, :, xs].copy(), B[:, ys][:, :, xs].copy())
            del E, B
    assert sim.counters()["particles"] == n0
    sim.close()
    o = oracle_run("C5")
    rec = {"config": "C5", "precision": precision, "continuity": cont, "patches": []}
    for k in range(len(F.C5_ORIGINS)):
        pr = {}
        for n in F.C5_SNAPS:
            Eg, Bg = (a[:, m:W - m, m:W - m] for a in got[(k, n)])
            Eo, Bo = (o["p%d_%s%d" % (k, w, n)][:, m:W - m, m:W - m] for w in "EB")
            feg = 0.5 * dx * dy * float(np.sum(Eg.astype(np.float64) ** 2) + np.sum(Bg.astype(np.float64) ** 2))
            feo = 0.5 * dx * dy * float(np.sum(Eo ** 2) + np.sum(Bo ** 2))
            pr[n] = {"E_rel_l2": rel_l2(Eg, Eo), "B_rel_l2": rel_l2(Bg, Bo), "fe_rel": abs(feg - feo) / feo}
        rec["patches"].append(pr)
    _report("C5_%s" % precision, rec)
    assert max(r for _, r in cont) <= CONT_TOL, rec
    for pr in rec["patches"]:
        assert pr[10]["E_rel_l2"] <= FIELD_TOL and pr[10]["B_rel_l2"] <= FIELD_TOL, pr
        assert all(pr[n]["fe_rel"] <= ENERGY_TOL for n in F.C5_SNAPS), pr
        assert pr[F.C5_STEPS]["E_rel_l2"] <= FINAL_E_TOL and pr[F.C5_STEPS]["B_rel_l2"] <= FINAL_B_TOL, pr
