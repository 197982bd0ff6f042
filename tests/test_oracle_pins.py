"""Pins of the fp64 oracle against what the paper and the mathematics fix (SURVEY.md §8(c)
P1-P13).  None of these re-types the oracle's formulas: they check closed forms, exact
discrete identities of the scheme, textbook library routines (scipy / numpy) and the paper's
worked values in tests/golden/.  CPU only."""
import json
import math
import os

import numpy as np
import pytest

from oracle import lib as L
from oracle.sim import OracleSim

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))
STAG = {"Ex": (0.5, 0.0), "Ey": (0.0, 0.5), "Ez": (0.0, 0.0), "Bx": (0.0, 0.5), "By": (0.5, 0.0), "Bz": (0.5, 0.5)}
ORDER = ["Ex", "Ey", "Ez", "Bx", "By", "Bz"]


def _rand_particles(rng, n, nx, ny, margin=0):
    ix = rng.integers(margin, nx - margin, n).astype(np.int32)
    iy = rng.integers(margin, ny - margin, n).astype(np.int32)
    x = rng.random(n)
    y = rng.random(n)
    return ix, iy, x, y


def _fill_periodic(F_interior, bcx=0, bcy=0, is_E=True):
    """(3, ny, nx) interior -> guard-extended grid with periodic guards (via the oracle's guard
    refresh; the guard refresh itself is pinned in test_guard_refresh_periodic)."""
    ny, nx = F_interior.shape[1:]
    G = L.grid(nx, ny)
    G[:, 1:ny + 1, 1:nx + 1] = F_interior
    L.refresh_guards(G, bcx, bcy, is_E)
    return G


# ---------------------------------------------------------------------------------------
# P1 gather ("bi-linear interpolation")
def test_guard_refresh_periodic():
    rng = np.random.default_rng(1)
    A = rng.random((3, 5, 7))
    G = _fill_periodic(A)
    ext = np.pad(A, ((0, 0), (1, 2), (1, 2)), mode="wrap")    # numpy's own periodic padding
    assert np.array_equal(G, ext)


def test_interp_constant_and_golden():
    nx, ny = 6, 5
    E = _fill_periodic(np.broadcast_to(np.array([1.0, 2.0, 3.0])[:, None, None], (3, ny, nx)).copy())
    B = _fill_periodic(np.broadcast_to(np.array([4.0, 5.0, 6.0])[:, None, None], (3, ny, nx)).copy(), is_E=False)
    rng = np.random.default_rng(2)
    ix, iy, x, y = _rand_particles(rng, 50, nx, ny)
    Ep, Bp = L.interpolate(E, B, ix, iy, x, y)
    assert np.allclose(Ep, [1, 2, 3], atol=4e-15, rtol=0)
    assert np.allclose(Bp, [4, 5, 6], atol=8e-15, rtol=0)
    # SPEC.md:133 worked example: Ez(x, y) = x (cell units, unstaggered) at ix=3, x=0.25 -> 3.25
    g = GOLD["interp_affine_ez"]
    nx, ny = 8, 8
    Ez = np.zeros((3, ny, nx))
    Ez[2] = np.arange(nx)[None, :]
    G = L.grid(nx, ny)
    G[:, 1:ny + 1, 1:nx + 1] = Ez
    G[2, :, 0] = -1.0
    G[2, :, nx + 1] = nx
    G[2, :, nx + 2] = nx + 1
    G[2, 0, :] = G[2, 1, :]
    G[2, ny + 1:, :] = G[2, ny, :]
    Ep, _ = L.interpolate(G, L.grid(nx, ny), np.array([g["ix"]], np.int32), np.array([g["iy"]], np.int32),
                          np.array([g["x"]]), np.array([g["y"]]))
    assert Ep[0, 2] == pytest.approx(g["expected_ez"], abs=1e-15)


def test_interp_affine_all_staggerings():
    """Bilinear interpolation is exact on affine fields F = a + b X + c Y sampled at each
    component's own staggered nodes; a wrong stagger offset is off by b/2."""
    nx, ny = 12, 10
    rng = np.random.default_rng(3)
    coef = rng.normal(size=(6, 3))
    grids = []
    for k, name in enumerate(ORDER):
        sx, sy = STAG[name]
        i = np.arange(-1, nx + 2)[None, :]
        j = np.arange(-1, ny + 2)[:, None]
        grids.append(coef[k, 0] + coef[k, 1] * (i + sx) + coef[k, 2] * (j + sy))
    E = np.ascontiguousarray(np.stack(grids[:3]))
    B = np.ascontiguousarray(np.stack(grids[3:]))
    ix, iy, x, y = _rand_particles(rng, 300, nx, ny, margin=1)
    x[:10] = 0.5
    x[10:20] = 0.0
    y[20:30] = 0.5
    Ep, Bp = L.interpolate(E, B, ix, iy, x, y)
    X, Y = ix + x, iy + y
    for k in range(6):
        want = coef[k, 0] + coef[k, 1] * X + coef[k, 2] * Y
        got = (Ep if k < 3 else Bp)[:, k % 3]
        assert np.max(np.abs(got - want)) < 1e-12, ORDER[k]


def test_interp_vs_scipy_map_coordinates():
    """Textbook routine: order-1 spline interpolation with periodic wrap on random fields."""
    from scipy.ndimage import map_coordinates
    nx, ny = 9, 7
    rng = np.random.default_rng(4)
    A = rng.normal(size=(3, ny, nx))
    Bi = rng.normal(size=(3, ny, nx))
    E = _fill_periodic(A)
    B = _fill_periodic(Bi, is_E=False)
    ix, iy, x, y = _rand_particles(rng, 400, nx, ny)
    Ep, Bp = L.interpolate(E, B, ix, iy, x, y)
    X, Y = ix + x, iy + y
    for k, name in enumerate(ORDER):
        sx, sy = STAG[name]
        arr = (A if k < 3 else Bi)[k % 3]
        want = map_coordinates(arr, [Y - sy, X - sx], order=1, mode="grid-wrap")
        got = (Ep if k < 3 else Bp)[:, k % 3]
        assert np.max(np.abs(got - want)) < 1e-13, name


# ---------------------------------------------------------------------------------------
# P2 Boris
def test_boris_force_free_and_e_kick():
    rng = np.random.default_rng(5)
    u = rng.normal(size=(3, 64)) * 2
    ux, uy, uz = (np.ascontiguousarray(u[i].copy()) for i in range(3))
    L.boris(ux, uy, uz, np.zeros((64, 3)), np.zeros((64, 3)), -1.0, 0.07)
    assert np.array_equal(np.stack([ux, uy, uz]), u)
    # E only: Delta u = (q/m) E dt = E dt / m_q exactly (two half kicks)
    E0 = rng.normal(size=(64, 3))
    ux, uy, uz = (np.ascontiguousarray(u[i].copy()) for i in range(3))
    L.boris(ux, uy, uz, E0, np.zeros((64, 3)), -2.0, 0.05)
    assert np.allclose(np.stack([ux, uy, uz]).T - u.T, E0 * 0.05 / -2.0, atol=1e-14, rtol=0)


def test_boris_rotation_angle_and_norm():
    """E = 0, uniform B: |u| conserved; rotation angle per step = 2 atan(|q/m| B dt / (2 gamma))
    about B."""
    rng = np.random.default_rng(6)
    n = 200
    u = rng.normal(size=(3, n)) * rng.uniform(0.01, 10, size=n)
    Bv = rng.normal(size=(n, 3)) * rng.uniform(0.1, 20, size=(n, 1))
    m_q, dt = -1.0, 0.07
    ux, uy, uz = (np.ascontiguousarray(u[i].copy()) for i in range(3))
    L.boris(ux, uy, uz, np.zeros((n, 3)), Bv, m_q, dt)
    un = np.stack([ux, uy, uz])
    assert np.allclose(np.linalg.norm(un, axis=0), np.linalg.norm(u, axis=0), rtol=1e-14)
    g = np.sqrt(1 + np.sum(u * u, axis=0))
    bhat = Bv.T / np.linalg.norm(Bv, axis=1)
    theta = 2 * np.arctan(np.linalg.norm(Bv, axis=1) * dt / (2 * g * abs(m_q)))
    # component perpendicular to B rotates by theta; parallel component unchanged
    upar0 = np.sum(u * bhat, axis=0)
    upar1 = np.sum(un * bhat, axis=0)
    assert np.allclose(upar0, upar1, atol=1e-12)
    p0 = u - upar0 * bhat
    p1 = un - upar1 * bhat
    cosang = np.sum(p0 * p1, axis=0) / (np.linalg.norm(p0, axis=0) * np.linalg.norm(p1, axis=0))
    sinang = np.sum(np.cross(p0.T, p1.T).T * bhat, axis=0) / (np.linalg.norm(p0, axis=0) * np.linalg.norm(p1, axis=0))
    ang = np.arctan2(sinang, cosang)
    # electrons (q < 0) gyrate counter-clockwise about B: rotation by +theta
    assert np.allclose(ang, theta * np.sign(-m_q), atol=1e-12)


def test_gyration_circle():
    """Full particle advance in a uniform Bz, E = 0: positions lie on a circle of radius
    R = v dt / (2 sin(theta/2)), and successive displacements turn by theta."""
    nx = ny = 64
    dx = dy = 0.1
    dt, m_q, B0 = 0.07, -1.0, 3.0
    E = L.grid(nx, ny)
    B = L.grid(nx, ny)
    B[2] = B0
    ix, iy = np.array([32], np.int32), np.array([32], np.int32)
    x, y = np.array([0.3]), np.array([0.6])
    ux, uy, uz = np.array([0.4]), np.array([0.0]), np.array([0.0])
    J = L.grid(nx, ny)
    pts = []
    for _ in range(60):
        Ep, Bp = L.interpolate(E, B, ix, iy, x, y)
        L.boris(ux, uy, uz, Ep, Bp, m_q, dt)
        L.advance_deposit(ix, iy, x, y, ux, uy, uz, -1.0, dt, dx, dy, J)
        pts.append(((ix[0] + x[0]) * dx, (iy[0] + y[0]) * dy))
    P = np.array(pts)
    g = math.sqrt(1 + 0.4 ** 2)
    v = 0.4 / g
    theta = 2 * math.atan(B0 * dt / (2 * g))
    R = v * dt / (2 * math.sin(theta / 2))
    d = np.diff(P, axis=0)
    turn = np.arctan2(d[1:, 1] * d[:-1, 0] - d[1:, 0] * d[:-1, 1], np.sum(d[1:] * d[:-1], axis=1))
    assert np.allclose(np.abs(turn), theta, atol=1e-11)
    # circumcentre of three points, then every point at distance R
    (ax, ay), (bx, by), (cx, cy) = P[0], P[7], P[15]
    D = 2 * (ax * (by - cy) + bx * (cy - ay) + cx * (ay - by))
    ux_ = ((ax ** 2 + ay ** 2) * (by - cy) + (bx ** 2 + by ** 2) * (cy - ay) + (cx ** 2 + cy ** 2) * (ay - by)) / D
    uy_ = ((ax ** 2 + ay ** 2) * (cx - bx) + (bx ** 2 + by ** 2) * (ax - cx) + (cx ** 2 + cy ** 2) * (bx - ax)) / D
    r = np.hypot(P[:, 0] - ux_, P[:, 1] - uy_)
    assert np.allclose(r, R, atol=1e-11)


# ---------------------------------------------------------------------------------------
# P3 / P4 deposit ("exact charge conserving method")
def _rho(nx, ny, q, ix, iy, x, y):
    """Independent node charge: area weights (1-x)(1-y) ... on the 4 nodes of the cell, periodic."""
    r = np.zeros((ny, nx))
    ix = np.mod(ix, nx)
    iy = np.mod(iy, ny)
    for (a, b, w) in ((0, 0, (1 - x) * (1 - y)), (1, 0, x * (1 - y)), (0, 1, (1 - x) * y), (1, 1, x * y)):
        np.add.at(r, ((iy + b) % ny, (ix + a) % nx), q * w)
    return r


def _divJ(J, nx, ny, dx, dy):
    Jx = J[0, 1:ny + 1, 1:nx + 1]
    Jy = J[1, 1:ny + 1, 1:nx + 1]
    return (Jx - np.roll(Jx, 1, axis=1)) / dx + (Jy - np.roll(Jy, 1, axis=0)) / dy


def test_deposit_no_motion_zero_current():
    nx = ny = 6
    rng = np.random.default_rng(7)
    ix, iy, x, y = _rand_particles(rng, 20, nx, ny)
    z = np.zeros(20)
    J = L.grid(nx, ny)
    L.advance_deposit(ix, iy, x, y, z.copy(), z.copy(), z.copy(), 0.5, 0.07, 0.1, 0.1, J)
    assert not np.any(J)


def test_deposit_pure_x_flux_sum():
    """Single-cell x motion: sum of jx = q Dx dx/dt, jy = 0."""
    nx = ny = 6
    dt, dx, dy, q = 0.07, 0.1, 0.1, -0.3
    J = L.grid(nx, ny)
    ix, iy = np.array([2], np.int32), np.array([3], np.int32)
    x, y = np.array([0.2]), np.array([0.35])
    ux = np.array([0.5])
    L.advance_deposit(ix, iy, x, y, ux, np.zeros(1), np.zeros(1), q, dt, dx, dy, J)
    Dx = 0.5 / math.sqrt(1.25) * dt / dx
    assert np.sum(J[0]) == pytest.approx(q * Dx * dx / dt, rel=1e-14)
    assert np.max(np.abs(J[1])) == 0.0
    assert x[0] == pytest.approx(0.2 + Dx, abs=1e-15) and ix[0] == 2


@pytest.mark.parametrize("seed", [8, 9, 10])
def test_deposit_discrete_continuity(seed):
    """rho^{n+1} - rho^n + dt div J = 0 at every node, for random <= 1-cell moves including
    corner and double crossings (north star: 1e-12)."""
    nx, ny, dx, dy, dt = 8, 7, 0.1, 0.13, 0.07
    rng = np.random.default_rng(seed)
    n = 3000
    ix, iy, x, y = _rand_particles(rng, n, nx, ny)
    x[:100] = 0.0           # exactly on an edge
    y[100:200] = 0.0
    x[200:300] = 1 - 1e-12  # next to an edge
    u = rng.normal(size=(3, n)) * 4.0
    q = -0.25
    rho0 = _rho(nx, ny, q, ix, iy, x, y)
    J = L.grid(nx, ny)
    bad = L.advance_deposit(ix, iy, x, y, u[0].copy(), u[1].copy(), u[2].copy(), q, dt, dx, dy, J)
    assert bad == 0
    assert np.all((x >= 0) & (x < 1) & (y >= 0) & (y < 1))
    L.fold_current(J, 0, 0)
    rho1 = _rho(nx, ny, q, ix, iy, x, y)
    res = rho1 - rho0 + dt * _divJ(J, nx, ny, dx, dy)
    assert np.max(np.abs(res)) < 1e-12


def test_deposit_jz_quadrature_and_sum():
    """Jz equals q vz (1/T) int S(x(t), y(t)) dt (bilinear S) by fine midpoint quadrature, and
    sums to q vz."""
    nx = ny = 6
    dt, dx, dy, q = 0.07, 0.1, 0.1, 0.7
    rng = np.random.default_rng(11)
    for trial in range(40):
        ix, iy = np.array([2], np.int32), np.array([2], np.int32)
        x0, y0 = rng.random(), rng.random()
        u = rng.normal(size=3) * 3
        J = L.grid(nx, ny)
        x, y = np.array([x0]), np.array([y0])
        L.advance_deposit(ix, iy, x, y, np.array([u[0]]), np.array([u[1]]), np.array([u[2]]), q, dt, dx, dy, J)
        g = math.sqrt(1 + u @ u)
        Dx, Dy, vz = u[0] / g * dt / dx, u[1] / g * dt / dy, u[2] / g
        M = 4000
        t = (np.arange(M) + 0.5) / M
        X = 2 + x0 + t * Dx
        Y = 2 + y0 + t * Dy
        want = np.zeros((ny + 3, nx + 3))
        i0 = np.floor(X).astype(int)
        j0 = np.floor(Y).astype(int)
        wx, wy = X - i0, Y - j0
        for a in (0, 1):
            for b in (0, 1):
                np.add.at(want, (j0 + b + 1, i0 + a + 1), ((wx if a else 1 - wx) * (wy if b else 1 - wy)) / M)
        want *= q * vz
        assert np.max(np.abs(J[2] - want)) < 2e-7 * abs(q * vz) + 1e-15
        assert np.sum(J[2]) == pytest.approx(q * vz, rel=1e-13, abs=1e-15)


def test_fold_periodic_equals_wrapped_deposit():
    """Ghost reduction: after the fold, the interior equals the deposit of the
    same particles with periodic wrap of every node index."""
    nx, ny = 5, 4
    rng = np.random.default_rng(12)
    J = L.grid(nx, ny)
    J[:] = rng.normal(size=J.shape)
    want = np.zeros((3, ny, nx))
    for jj in range(-1, ny + 2):
        for ii in range(-1, nx + 2):
            want[:, jj % ny, ii % nx] += J[:, jj + 1, ii + 1]
    L.fold_current(J, 0, 0)
    assert np.allclose(J[:, 1:ny + 1, 1:nx + 1], want, atol=1e-14)
    assert np.array_equal(J, np.pad(J[:, 1:ny + 1, 1:nx + 1], ((0, 0), (1, 2), (1, 2)), mode="wrap"))
    J2 = L.grid(nx, ny)
    J2[:] = rng.normal(size=J2.shape)
    inner = J2[:, 1:ny + 1, 1:nx + 1].copy()
    L.fold_current(J2, 1, 1)   # open: guard contributions discarded
    assert np.array_equal(J2[:, 1:ny + 1, 1:nx + 1], inner)
    assert not np.any(J2[:, 0, :]) and not np.any(J2[:, :, -2:])


# ---------------------------------------------------------------------------------------
# P5 whole loop: Gauss's law and div B are constants of the discrete scheme
def _divE(E, nx, ny, dx, dy):
    Ex = E[0, 1:ny + 1, 1:nx + 1]
    Ey = E[1, 1:ny + 1, 1:nx + 1]
    return (Ex - np.roll(Ex, 1, axis=1)) / dx + (Ey - np.roll(Ey, 1, axis=0)) / dy


def _divB(B, nx, ny, dx, dy):
    """div B at the cell centres (i+1/2, j+1/2)."""
    Bx = B[0, 1:ny + 1, 1:nx + 1]
    By = B[1, 1:ny + 1, 1:nx + 1]
    return (np.roll(Bx, -1, axis=1) - Bx) / dx + (np.roll(By, -1, axis=0) - By) / dy


def test_gauss_law_and_divb_preserved():
    nx, ny, dx, dy, dt = 8, 6, 0.1, 0.12, 0.06
    rng = np.random.default_rng(13)
    sp = []
    for m_q, n in ((-1.0, 1.0), (1.0, 1.0)):
        N = nx * ny * 4
        ix, iy, x, y = _rand_particles(rng, N, nx, ny)
        u = rng.normal(size=(3, N)) * 0.3
        sp.append(dict(m_q=m_q, n=n, ppc=(2, 2), ufl=(0, 0, 0), uth=(0, 0, 0), ix=ix, iy=iy, x=x, y=y,
                       ux=u[0], uy=u[1], uz=u[2]))
    sim = OracleSim(nx, ny, dx, dy, dt, sp)

    def gauss():
        rho = sum(_rho(nx, ny, s["q"], s["ix"], s["iy"], s["x"], s["y"]) for s in sim.species)
        return _divE(sim.E, nx, ny, dx, dy) - rho
    g0 = gauss()
    for _ in range(60):
        sim.step()
    assert np.max(np.abs(gauss() - g0)) < 1e-12
    assert np.max(np.abs(_divB(sim.B, nx, ny, dx, dy))) < 1e-12
    assert np.max(np.abs(sim.E)) > 1e-3      # non-trivial dynamics


# ---------------------------------------------------------------------------------------
# P6 Yee vacuum ("FDTD ... on a Yee mesh")
def _dispersion_cos(kx, ky, dx, dy, dt):
    K2 = (2 / dx * math.sin(kx * dx / 2)) ** 2 + (2 / dy * math.sin(ky * dy / 2)) ** 2
    return 1 - dt * dt * K2 / 2


@pytest.mark.parametrize("mode", ["TM", "TE"])
def test_yee_dispersion(mode):
    """Single eigenmode: cos(omega dt) from the 3-term estimator equals the Yee closed form
    sin(omega dt/2)/dt = sqrt((sin(kx dx/2)/dx)^2 + (sin(ky dy/2)/dy)^2)."""
    nx, ny, dx, dy, dt = 16, 12, 0.1, 0.13, 0.06
    mx, my = 3, 2
    kx, ky = 2 * math.pi * mx / (nx * dx), 2 * math.pi * my / (ny * dy)
    E = L.grid(nx, ny)
    B = L.grid(nx, ny)
    i = np.arange(nx)[None, :]
    j = np.arange(ny)[:, None]
    if mode == "TM":
        E[2, 1:ny + 1, 1:nx + 1] = np.cos(kx * i * dx + ky * j * dy)
        comp, F = 2, E
    else:
        B[2, 1:ny + 1, 1:nx + 1] = np.cos(kx * (i + 0.5) * dx + ky * (j + 0.5) * dy)
        comp, F = 2, B
    L.refresh_guards(E, 0, 0, True)
    L.refresh_guards(B, 0, 0, False)
    J = L.grid(nx, ny)
    series = [F[comp, 1:ny + 1, 1:nx + 1].copy()]
    for _ in range(120):
        L.yee_advance(E, B, J, dt, dx, dy, 0, 0)
        series.append(F[comp, 1:ny + 1, 1:nx + 1].copy())
    S = np.array(series)
    num = np.sum(S[1:-1] * (S[2:] + S[:-2]))
    den = 2 * np.sum(S[1:-1] ** 2)
    assert num / den == pytest.approx(_dispersion_cos(kx, ky, dx, dy, dt), abs=1e-13)


def _curlE(E, nx, ny, dx, dy):
    """curl E at the B points (numpy rolls on periodic interiors)."""
    Ex, Ey, Ez = (E[c, 1:ny + 1, 1:nx + 1] for c in range(3))
    cx = (np.roll(Ez, -1, 0) - Ez) / dy
    cy = -(np.roll(Ez, -1, 1) - Ez) / dx
    cz = (np.roll(Ey, -1, 1) - Ey) / dx - (np.roll(Ex, -1, 0) - Ex) / dy
    return np.stack([cx, cy, cz])


def test_yee_exact_invariant_and_travelling_wave_energy():
    """Vacuum, J = 0: W = 1/2 sum(E^n.E^n + B^{n-1/2}.B^{n+1/2}), B^{n-+1/2} = B^n +- (dt/2) curl E^n,
    is conserved exactly."""
    nx, ny, dx, dy, dt = 16, 16, 0.1, 0.1, 0.06
    rng = np.random.default_rng(14)
    E = L.grid(nx, ny)
    B = L.grid(nx, ny)
    E[:, 1:ny + 1, 1:nx + 1] = rng.normal(size=(3, ny, nx))
    B[:, 1:ny + 1, 1:nx + 1] = rng.normal(size=(3, ny, nx))
    L.refresh_guards(E, 0, 0, True)
    L.refresh_guards(B, 0, 0, False)
    J = L.grid(nx, ny)

    def W():
        Bi = B[:, 1:ny + 1, 1:nx + 1]
        c = _curlE(E, nx, ny, dx, dy)
        Bm, Bp = Bi + 0.5 * dt * c, Bi - 0.5 * dt * c
        return 0.5 * (np.sum(E[:, 1:ny + 1, 1:nx + 1] ** 2) + np.sum(Bm * Bp))
    w0 = W()
    for _ in range(200):
        L.yee_advance(E, B, J, dt, dx, dy, 0, 0)
    assert W() == pytest.approx(w0, rel=1e-12)


# ---------------------------------------------------------------------------------------
# P7 filter ("compensated binomial filter")
def test_filter_pass_is_circular_convolution_and_transfer():
    nx, ny = 24, 5
    rng = np.random.default_rng(15)
    A = rng.normal(size=(3, ny, nx))
    J = _fill_periodic(A)
    L.filter_x(J, 0, 0, 1, False)
    k = np.array([0.25, 0.5, 0.25])
    want = np.stack([np.stack([np.convolve(np.concatenate([r[-1:], r, r[:1]]), k, mode="valid") for r in c]) for c in A])
    assert np.allclose(J[:, 1:ny + 1, 1:nx + 1], want, atol=1e-15)
    # impulse -> (1/4, 1/2, 1/4) (golden)
    J = L.grid(nx, ny)
    J[0, 3, 10] = 1.0
    L.refresh_guards(J, 0, 0, False)
    L.filter_x(J, 0, 0, 1, False)
    assert np.allclose(J[0, 3, 9:12], GOLD["filter_impulse"]["expected"], atol=0)
    # single Fourier modes: T(k) = cos^{2n}(k dx/2) (1 + n sin^2(k dx/2)) with the compensator
    for n in (1, 2, 4):
        for m in (0, 1, 5, 12):
            kk = 2 * math.pi * m / nx
            row = np.cos(kk * np.arange(nx))
            J = _fill_periodic(np.broadcast_to(row, (3, ny, nx)).copy())
            L.filter_x(J, 0, 0, n, True)
            T = math.cos(kk / 2) ** (2 * n) * (1 + n * math.sin(kk / 2) ** 2)
            assert np.allclose(J[:, 1:ny + 1, 1:nx + 1], T * row, atol=1e-14)
    # Nyquist is annihilated by a binomial pass; DC preserved
    J = _fill_periodic(np.broadcast_to((-1.0) ** np.arange(nx), (3, ny, nx)).copy())
    L.filter_x(J, 0, 0, 1, False)
    assert np.max(np.abs(J)) < 1e-15


# ---------------------------------------------------------------------------------------
# P8 cold plasma oscillation (k = 0)
def test_cold_plasma_frequency():
    g = GOLD["cold_plasma_omega"]
    nx = ny = 4
    dx = dy = 0.1
    dt = g["dt"]
    N = nx * ny * 4
    l, k = np.divmod(np.arange(4), 2)
    ix = np.repeat(np.arange(nx * ny) % nx, 4).astype(np.int32)
    iy = np.repeat(np.arange(nx * ny) // nx, 4).astype(np.int32)
    sp = [dict(m_q=-1.0, n=1.0, ppc=(2, 2), ufl=(0, 0, 0), uth=(0, 0, 0), ix=ix, iy=iy,
               x=np.tile((k + 0.5) / 2, nx * ny), y=np.tile((l + 0.5) / 2, nx * ny),
               ux=np.full(N, 1e-4), uy=np.zeros(N), uz=np.zeros(N))]
    sim = OracleSim(nx, ny, dx, dy, dt, sp)
    ex = []
    for _ in range(300):
        sim.step()
        ex.append(sim.E[0, 1:ny + 1, 1:nx + 1].copy())
    S = np.array(ex)
    assert np.ptp(S[-1]) < 1e-15 * max(1.0, np.max(np.abs(S)))     # spatially uniform
    s = S[:, 0, 0]
    c = np.sum(s[1:-1] * (s[2:] + s[:-2])) / (2 * np.sum(s[1:-1] ** 2))
    omega = math.acos(c) / dt
    assert omega == pytest.approx(g["omega"], rel=1e-7)
    assert omega == pytest.approx(2 / dt * math.asin(dt / 2), rel=1e-7)


def test_pair_plasma_frequency():
    """Positive charges (m_q = +1, the paper's positron cloud): a cold
    electron-positron plasma (n = 1 each) with the two species displaced in opposite directions
    oscillates at the total plasma frequency w_p^2 = sum_s n_s q_s^2 / m_s = 2, i.e. the Yee /
    leapfrog dispersion w = (2/dt) asin(sqrt(2) dt / 2); a sign error in the charge, the Boris
    factor or the deposit of m_q > 0 changes w (or makes the mode grow)."""
    nx = ny = 4
    dx = dy = 0.1
    dt = 0.07
    N = nx * ny * 4
    l, k = np.divmod(np.arange(4), 2)
    ix = np.repeat(np.arange(nx * ny) % nx, 4).astype(np.int32)
    iy = np.repeat(np.arange(nx * ny) // nx, 4).astype(np.int32)

    def sp(m_q, u0):
        return dict(m_q=m_q, n=1.0, ppc=(2, 2), ufl=(0, 0, 0), uth=(0, 0, 0), ix=ix.copy(), iy=iy.copy(),
                    x=np.tile((k + 0.5) / 2, nx * ny), y=np.tile((l + 0.5) / 2, nx * ny),
                    ux=np.full(N, u0), uy=np.zeros(N), uz=np.zeros(N))

    sim = OracleSim(nx, ny, dx, dy, dt, [sp(-1.0, 1e-4), sp(1.0, -1e-4)])
    ex = []
    for _ in range(300):
        sim.step()
        ex.append(sim.E[0, 1, 1])
    s_ = np.array(ex)
    c = np.sum(s_[1:-1] * (s_[2:] + s_[:-2])) / (2 * np.sum(s_[1:-1] ** 2))
    omega = math.acos(c) / dt
    assert omega == pytest.approx(2 / dt * math.asin(math.sqrt(2.0) * dt / 2), rel=1e-7)
    # the two species move in antiphase with equal and opposite momenta (equal mass, opposite charge)
    assert np.allclose(sim.species[0]["ux"], -sim.species[1]["ux"], atol=1e-18, rtol=1e-12)


# ---------------------------------------------------------------------------------------
# P9 Mur-1 open boundary
def test_mur_absorbs_normal_pulse():
    nx, ny, dx, dy, dt = 400, 4, 0.1, 0.1, 0.07
    E = L.grid(nx, ny)
    B = L.grid(nx, ny)
    i = np.arange(nx)
    xc, w = 20.0, 1.0
    E[1, 1:ny + 1, 1:nx + 1] = np.exp(-((i * dx - xc) / w) ** 2)[None, :]
    B[2, 1:ny + 1, 1:nx + 1] = np.exp(-(((i + 0.5) * dx - xc) / w) ** 2)[None, :]
    L.refresh_guards(E, 1, 0, True)
    L.refresh_guards(B, 1, 0, False)
    J = L.grid(nx, ny)
    e0 = L.field_energy(E, B, dx, dy)
    for _ in range(int(32 / dt)):
        L.yee_advance(E, B, J, dt, dx, dy, 1, 0)
    assert L.field_energy(E, B, dx, dy) / e0 < 1e-4


# ---------------------------------------------------------------------------------------
# P11 moving window
def test_window_shift_composition_injection_and_exit():
    nx, ny = 12, 5
    rng = np.random.default_rng(16)
    A = rng.normal(size=(3, ny, nx))
    sp = [dict(m_q=-1.0, n=1.0, ppc=(2, 2), ufl=(0, 0, 0), uth=(0, 0, 0), ix=np.array([0, 5], np.int32),
               iy=np.array([1, 2], np.int32), x=np.array([0.5, 0.5]), y=np.array([0.5, 0.5]), ux=np.zeros(2),
               uy=np.zeros(2), uz=np.zeros(2), id=np.array([0, 1]))]
    sim = OracleSim(nx, ny, 0.1, 0.1, 0.05, sp, bc=(2, 1), E=A, B=A)
    sim._shift_window()
    sim._shift_window()
    # two single shifts == one double shift: F'[i] = F[i+2], two fresh zero columns
    want = np.concatenate([A[:, :, 2:], np.zeros((3, ny, 2))], axis=2)
    assert np.array_equal(sim.fields(0), want) and np.array_equal(sim.fields(1), want)
    s = sim.species[0]
    for_ = [k for k in range(len(s["id"])) if s["id"][k] >= 2 ** 31]
    assert len(for_) == 2 * ny * 4                    # ppc * ny per shift
    assert len(set(s["id"][for_].tolist())) == len(for_)
    sim._particle_bc(s, window_now=True)             # the particle at ix = 0 left (ix = -2)
    assert 0 not in s["id"] and 1 in s["id"]
    assert s["ix"][list(s["id"]).index(1)] == 3


# ---------------------------------------------------------------------------------------
# P13 init (shared synth inputs) and energy conventions
def test_injection_counts_cold_and_determinism():
    import synth
    cfg = synth.config("C1", nx=8, ny=6)
    p = synth.species_particles(cfg, 0)
    assert len(p["ix"]) == 8 * 6 * 16
    assert len(np.unique(p["id"])) == len(p["id"])
    q = synth.species_particles(cfg, 0)
    for k in p:
        assert np.array_equal(p[k], q[k])
    cold = synth.config("C1", nx=4, ny=4)
    cold["species"][0]["uth"] = (0.0, 0.0, 0.0)
    c = synth.species_particles(cold, 0)
    assert not np.any(c["ux"]) and not np.any(c["uy"]) and not np.any(c["uz"])
    N = synth.normals(7, 0, np.arange(200000))
    assert abs(N.mean()) < 0.01 and abs(N.std() - 1) < 0.01
    c3 = synth.config("C3", nx=32, ny=4)
    c3["species"][1].update(x0=1.6, x1=3.2)
    slab = synth.species_particles(c3, 1)
    assert np.all(slab["ix"] >= 16) and len(slab["ix"]) == 16 * 4 * 8


def test_energy_conventions():
    """FE = 1/2 dx dy sum(E^2 + B^2); KE_s = q m_q dx dy sum(gamma- - 1) >= 0 (R8)."""
    nx = ny = 4
    dx, dy, dt = 0.1, 0.2, 0.05
    E = L.grid(nx, ny)
    B = L.grid(nx, ny)
    E[1, 1:ny + 1, 1:nx + 1] = 2.0
    B[0, 1:ny + 1, 1:nx + 1] = 1.0
    assert L.field_energy(E, B, dx, dy) == pytest.approx(0.5 * dx * dy * 16 * 5)
    u = np.array([0.3])
    sp = [dict(m_q=-1.0, n=1.0, ppc=(1, 1), ufl=(0, 0, 0), uth=(0, 0, 0), ix=np.array([1]), iy=np.array([1]),
               x=np.array([0.5]), y=np.array([0.5]), ux=u, uy=np.zeros(1), uz=np.zeros(1))]
    sim = OracleSim(nx, ny, dx, dy, dt, sp)
    sim.step()
    assert sim.ke[0][0] == pytest.approx(dx * dy * (math.sqrt(1 + 0.09) - 1), rel=1e-12)
    assert sim.fe[0] == 0.0


# ---------------------------------------------------------------------------------------
# P9 Mur-1 on y edges and with dx != dy (R13; C4 has dx = 0.02, dy = 0.1 and absorbing y edges)
def _pulse_energy_left(nx, ny, dx, dy, dt, bc, comp, axis, steps):
    E = L.grid(nx, ny)
    B = L.grid(nx, ny)
    if axis == "y":
        prof = np.exp(-((np.arange(ny) * dy - 0.5 * ny * dy) / 1.0) ** 2)[:, None]
    else:
        prof = np.exp(-((np.arange(nx) * dx - 0.5 * nx * dx) / 1.0) ** 2)[None, :]
    E[comp, 1:ny + 1, 1:nx + 1] = prof     # splits into two pulses running into both edges
    L.refresh_guards(E, *bc, True)
    L.refresh_guards(B, *bc, False)
    J = L.grid(nx, ny)
    e0 = L.field_energy(E, B, dx, dy)
    for _ in range(steps):
        L.yee_advance(E, B, J, dt, dx, dy, *bc)
    return L.field_energy(E, B, dx, dy) / e0


@pytest.mark.parametrize("comp", [0, 2])
def test_mur_y_edges_absorb_at_c4_spacing(comp):
    """A pulse of Ex (TE) or Ez (TM) running along y into both open y edges of a box with C4's
    cells (dx = 0.02, dy = 0.1, dt = 0.019): a first-order Mur boundary absorbs a smooth normally
    incident pulse to well below 1e-4 of its energy.  The y edges use kappa_y = (dt - dy)/(dt + dy);
    taking dx there instead leaves ~0.4 of the energy, so this pins the y branch."""
    left = _pulse_energy_left(4, 400, 0.02, 0.1, 0.019, (0, 1), comp, "y", int(30 / 0.019))
    assert left < 1e-4, left


@pytest.mark.parametrize("comp", [1, 2])
def test_mur_x_edges_absorb_with_unequal_cells(comp):
    """The same on the x edges with dy != dx (kappa_x = (dt - dx)/(dt + dx))."""
    left = _pulse_energy_left(400, 4, 0.1, 0.02, 0.019, (1, 0), comp, "x", int(30 / 0.019))
    assert left < 1e-4, left


def _open_box_state(nx, ny, rng):
    """Random E, B on every node an open-open box evolves (interior, plus the Mur node lines of
    tangential E at x = nx (Ey, Ez) and y = ny (Ex, Ez)); zero elsewhere."""
    E = L.grid(nx, ny)
    B = L.grid(nx, ny)
    E[0, 1:ny + 2, 1:nx + 1] = rng.normal(size=(ny + 1, nx))        # Ex: i < nx, j <= ny
    E[1, 1:ny + 1, 1:nx + 2] = rng.normal(size=(ny, nx + 1))        # Ey: i <= nx, j < ny
    E[2, 1:ny + 2, 1:nx + 2] = rng.normal(size=(ny + 1, nx + 1))    # Ez: i <= nx, j <= ny
    B[:, 1:ny + 1, 1:nx + 1] = rng.normal(size=(3, ny, nx))
    L.refresh_guards(E, 1, 1, True)
    L.refresh_guards(B, 1, 1, False)
    return E, B


def _mirror(E, B, nx, ny, axis):
    """The reflection x -> Lx - x (or y -> Ly - y) of a Yee state: node index i -> n - i,
    half-node index i -> n - 1 - i; E is a polar vector, B a pseudovector."""
    E2, B2 = np.zeros_like(E), np.zeros_like(B)
    n = nx if axis == "x" else ny
    def node(F, c, sign):       # index k of the axis (guard-extended position k + 1)
        src = F[c]
        dst = np.zeros_like(src)
        ax = 1 if axis == "x" else 0
        for k in range(0, n + 1):
            sl_d = [slice(None), slice(None)]; sl_s = [slice(None), slice(None)]
            sl_d[ax] = k + 1; sl_s[ax] = n - k + 1
            dst[tuple(sl_d)] = sign * src[tuple(sl_s)]
        return dst
    def half(F, c, sign):
        src = F[c]
        dst = np.zeros_like(src)
        ax = 1 if axis == "x" else 0
        for k in range(0, n):
            sl_d = [slice(None), slice(None)]; sl_s = [slice(None), slice(None)]
            sl_d[ax] = k + 1; sl_s[ax] = n - 1 - k + 1
            dst[tuple(sl_d)] = sign * src[tuple(sl_s)]
        return dst
    if axis == "x":   # x-staggered: Ex, By, Bz; polar flips Ex; pseudo flips By, Bz
        E2[0], E2[1], E2[2] = half(E, 0, -1), node(E, 1, 1), node(E, 2, 1)
        B2[0], B2[1], B2[2] = node(B, 0, 1), half(B, 1, -1), half(B, 2, -1)
    else:             # y-staggered: Ey, Bx, Bz; polar flips Ey; pseudo flips Bx, Bz
        E2[0], E2[1], E2[2] = node(E, 0, 1), half(E, 1, -1), node(E, 2, 1)
        B2[0], B2[1], B2[2] = half(B, 0, -1), node(B, 1, 1), half(B, 2, -1)
    return E2, B2


@pytest.mark.parametrize("axis", ["x", "y"])
def test_open_box_mirror_symmetry_and_corner_rule(axis):
    """Maxwell's equations and R13 treat the low and high edge of an open axis alike, so the
    discrete evolution of an open-open box commutes with the reflection of the box: evolving
    the mirror image of a random state equals the mirror image of the evolved state, to
    roundoff.  This pins every Mur node line, the guard placement of the high edges and the
    corner rule (all four corner nodes of Ez take the y-edge Mur; a corner handled differently
    from its mirror breaks the symmetry).  B's normal component on the edge line (Bx at x = 0,
    By at y = 0) feeds only Mur-overwritten E nodes and has no mirror partner; it is excluded."""
    nx, ny, dx, dy, dt = 13, 11, 0.1, 0.08, 0.045
    rng = np.random.default_rng(21)
    E, B = _open_box_state(nx, ny, rng)
    Em, Bm = _mirror(E, B, nx, ny, axis)
    J = L.grid(nx, ny)
    for _ in range(40):
        L.yee_advance(E, B, J, dt, dx, dy, 1, 1)
        L.yee_advance(Em, Bm, J, dt, dx, dy, 1, 1)
    Er, Br = _mirror(E, B, nx, ny, axis)
    if axis == "x":
        Br[0, :, [1, nx + 1]] = Bm[0, :, [1, nx + 1]] = 0.0     # Bx on the x = 0 line and its image
    else:
        Br[1, [1, ny + 1], :] = Bm[1, [1, ny + 1], :] = 0.0     # By on the y = 0 line and its image
    scale = max(np.max(np.abs(Em)), np.max(np.abs(Bm)))
    assert np.max(np.abs(Em - Er)) <= 1e-12 * scale
    assert np.max(np.abs(Bm - Br)) <= 1e-12 * scale
    # the corner nodes carry field (they are advanced, not held)
    for (i, j) in ((0, 0), (nx, 0), (0, ny), (nx, ny)):
        assert E[2, j + 1, i + 1] != 0.0


# ---------------------------------------------------------------------------------------
# P7 filter with zero guards (C4: window x axis, R12/R14)
@pytest.mark.parametrize("bcx", [1, 2])
def test_filter_zero_guards_is_zero_padded_convolution(bcx):
    nx, ny = 23, 4
    rng = np.random.default_rng(22)
    A = rng.normal(size=(3, ny, nx))
    for n, comp in ((1, False), (4, True)):
        J = L.grid(nx, ny)
        J[:, 1:ny + 1, 1:nx + 1] = A
        L.refresh_guards(J, bcx, 0, False)
        L.filter_x(J, bcx, 0, n, comp)
        want = A.copy()
        kernels = [np.array([0.25, 0.5, 0.25])] * n
        if comp:
            kernels.append(np.array([-n / 4, 1 + n / 2, -n / 4]))
        for k in kernels:   # numpy's own convolution of each row, zero outside the box
            want = np.stack([np.stack([np.convolve(r, k, mode="same") for r in c]) for c in want])
        assert np.allclose(J[:, 1:ny + 1, 1:nx + 1], want, rtol=0, atol=1e-14)


# ---------------------------------------------------------------------------------------
# a5 particle removal on open edges (C3 x, C4 y)
@pytest.mark.parametrize("axis", ["x", "y"])
def test_open_edge_removal_counts(axis):
    """Particles near both open edges of an axis, drifting at known speeds in a field-free box:
    exactly those whose straight path X + u/gamma dt/d leaves [0, n) are removed after one step,
    and the survivors keep their ids."""
    nx, ny, dx, dy, dt = 16, 12, 0.1, 0.08, 0.05
    rng = np.random.default_rng(23)
    N = 400
    n, d = (nx, dx) if axis == "x" else (ny, dy)
    lo = rng.random(N) < 0.5
    cell = np.where(lo, 0, n - 1).astype(np.int32)
    off = rng.random(N)
    u = rng.uniform(0.05, 3.0, N) * np.where(lo, -1.0, 1.0)   # outward at both edges
    u[rng.random(N) < 0.25] *= -1.0                             # some move inward
    other = rng.integers(2, (ny if axis == "x" else nx) - 2, N).astype(np.int32)
    z = np.zeros(N)
    sp = dict(m_q=-1.0, n=1.0, ppc=(1, 1), ufl=(0, 0, 0), uth=(0, 0, 0), id=np.arange(N),
              ix=cell if axis == "x" else other, iy=other if axis == "x" else cell,
              x=off if axis == "x" else rng.random(N), y=rng.random(N) if axis == "x" else off,
              ux=u if axis == "x" else z, uy=z if axis == "x" else u, uz=z)
    bc = (1, 0) if axis == "x" else (0, 1)
    sim = OracleSim(nx, ny, dx, dy, dt, [sp], bc=bc)
    X = cell + off + u / np.sqrt(1 + u * u) * dt / d
    gone = (X < 0) | (X >= n)
    assert 0 < np.count_nonzero(gone) < N
    sim.step()
    s = sim.species[0]
    assert np.array_equal(np.sort(s["id"]), np.arange(N)[~gone])


def test_window_injection_follows_the_profile_beyond_the_box():
    """R15: the entering column takes the species' density beyond the box: the
    ppc lattice for n > 0 (uniform, or a ramp that ends inside the box), nothing for n = 0; a slab
    profile or a ramp reaching past the box is rejected."""
    nx, ny = 10, 3
    base = dict(m_q=-1.0, ppc=(2, 1), ufl=(0, 0, 0), uth=(0, 0, 0), ix=np.zeros(0, np.int32),
                iy=np.zeros(0, np.int32), x=np.zeros(0), y=np.zeros(0), ux=np.zeros(0), uy=np.zeros(0),
                uz=np.zeros(0), id=np.zeros(0, np.int64))
    sps = [dict(base, n=1.0), dict(base, n=0.0), dict(base, n=2.0, profile="ramp", x0=0.2, x1=0.6)]
    sim = OracleSim(nx, ny, 0.1, 0.1, 0.05, sps, bc=(2, 1))
    sim._shift_window()
    assert [len(s["ix"]) for s in sim.species] == [2 * ny, 0, 2 * ny]
    assert np.all(sim.species[2]["ix"] == nx - 1)
    for bad in (dict(base, n=1.0, profile="slab", x0=0.0, x1=0.5), dict(base, n=1.0, profile="ramp", x0=0.5, x1=1.5)):
        sim = OracleSim(nx, ny, 0.1, 0.1, 0.05, [bad], bc=(2, 1))
        with pytest.raises(ValueError):
            sim._shift_window()


def test_cell_index_exemption_is_per_axis():
    """R23: an index mismatch is excused only when the oracle's offset is within 2^-20 of a cell
    edge on the mismatching axis (parity_util.compare_particles)."""
    from parity_util import compare_particles
    o = {"ix": np.array([3, 3, 3]), "iy": np.array([5, 5, 5]), "x": np.array([1e-9, 0.5, 0.5]),
         "y": np.array([0.5, 1e-9, 0.5]), "ux": np.zeros(3), "uy": np.zeros(3), "uz": np.zeros(3),
         "id": np.arange(3)}
    g = dict(o)
    g["ix"] = np.array([2, 2, 3])   # particle 0: x near its edge (excused); particle 1: y near, x differs
    g["iy"] = np.array([5, 5, 5])
    c = compare_particles(g, o, 16, 16)
    assert c["cell_bad"] == 1
