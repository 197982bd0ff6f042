"""Comparison helpers for the GPU-vs-oracle parity tests (tolerances: BASELINE.json north_star
and SURVEY.md §8(c) R19-R23).  CPU-only numpy; imports neither side's arithmetic."""
import numpy as np

POS_TOL = 1e-5        # R19: position error in cells, after 1 step
MOM_TOL = 1e-5        # R19: relative momentum error, after 1 step
FIELD_TOL = 1e-4      # R20: relative L2 of E and B after 10 steps
CONT_TOL = 1e-5       # R21: continuity residual / rho_ref
ENERGY_TOL = 0.01     # R22: energy histories within 1 % of the max
CELL_FRAC = 0.9999    # R23: bit-exact cell index fraction


def by_id(p):
    o = np.argsort(p["id"], kind="stable")
    return {k: np.asarray(v)[o] for k, v in p.items()}


def oracle_particles(sim, s):
    sp = sim.species[s]
    return {"ix": sp["ix"], "iy": sp["iy"], "x": sp["x"], "y": sp["y"], "ux": sp["ux"], "uy": sp["uy"],
            "uz": sp["uz"], "id": sp["id"].astype(np.uint64)}


def compare_particles(g, o, nx, ny, periodic=(True, True)):
    """Per-particle errors keyed by id (R19) and the cell-index agreement class (R23)."""
    g, o = by_id(g), by_id(o)
    assert np.array_equal(g["id"].astype(np.uint64), o["id"].astype(np.uint64)), "particle id sets differ"
    Xg = g["ix"].astype(np.float64) + g["x"]
    Xo = o["ix"].astype(np.float64) + o["x"]
    Yg = g["iy"].astype(np.float64) + g["y"]
    Yo = o["iy"].astype(np.float64) + o["y"]
    dX = Xg - Xo
    dY = Yg - Yo
    if periodic[0]:
        dX = (dX + nx / 2) % nx - nx / 2
    if periodic[1]:
        dY = (dY + ny / 2) % ny - ny / 2
    pos = np.maximum(np.abs(dX), np.abs(dY))
    ug = np.stack([g["ux"], g["uy"], g["uz"]]).astype(np.float64)
    uo = np.stack([o["ux"], o["uy"], o["uz"]]).astype(np.float64)
    mom = np.linalg.norm(ug - uo, axis=0) / np.maximum(np.linalg.norm(uo, axis=0), 1e-6)
    same_x = g["ix"] == o["ix"]
    same_y = g["iy"] == o["iy"]
    same = same_x & same_y
    # R23: a mismatch is a boundary-rounding case iff the oracle's offset is within 2^-20 of 0 or 1
    # on the axis that mismatches (each mismatching axis must be near its edge)
    eps = 2.0 ** -20
    near_x = np.minimum(o["x"], 1 - o["x"]) < eps
    near_y = np.minimum(o["y"], 1 - o["y"]) < eps
    excused = (same_x | near_x) & (same_y | near_y)
    bad_cells = np.count_nonzero(~same & ~excused)
    return {"pos_max": float(pos.max(initial=0.0)), "mom_max": float(mom.max(initial=0.0)),
            "cell_exact_frac": float(np.mean(same)) if len(same) else 1.0, "cell_bad": int(bad_cells), "n": len(same)}


def rel_l2(a, b):
    nb = np.linalg.norm(b.astype(np.float64))
    d = np.linalg.norm(a.astype(np.float64) - b.astype(np.float64))
    return d / nb if nb >= 1e-30 else d


def rho_nodes(nx, ny, q, p):
    """Node charge from particle positions: bilinear area weights, periodic wrap (R21)."""
    r = np.zeros((ny, nx))
    ix = np.mod(p["ix"], nx)
    iy = np.mod(p["iy"], ny)
    x = p["x"].astype(np.float64)
    y = p["y"].astype(np.float64)
    for a, b, w in ((0, 0, (1 - x) * (1 - y)), (1, 0, x * (1 - y)), (0, 1, (1 - x) * y), (1, 1, x * y)):
        np.add.at(r, ((iy + b) % ny, (ix + a) % nx), q * w)
    return r


def continuity_residual(nx, ny, dx, dy, dt, rho0, rho1, J, bc=(0, 0)):
    """max |rho1 - rho0 + dt div J| over nodes; cells within 2 of a non-periodic edge are
    excluded (R21: charge leaves there)."""
    Jx = J[0].astype(np.float64)
    Jy = J[1].astype(np.float64)
    div = (Jx - np.roll(Jx, 1, axis=1)) / dx + (Jy - np.roll(Jy, 1, axis=0)) / dy
    r = np.abs(rho1 - rho0 + dt * div)
    if bc[0] != 0:
        r = r[:, 2:-2]
    if bc[1] != 0:
        r = r[2:-2, :]
    return float(np.max(r))


def energy_agreement(hist_g, hist_o):
    """max |g(n) - o(n)| / max_m |o(m)| (R22)."""
    g = np.asarray(hist_g, dtype=np.float64)
    o = np.asarray(hist_o, dtype=np.float64)
    scale = np.max(np.abs(o))
    return float(np.max(np.abs(g - o)) / scale) if scale > 0 else float(np.max(np.abs(g - o)))
