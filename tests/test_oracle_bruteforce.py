"""Brute force (SURVEY.md §8(c) "Brute force"): one full oracle step for 1-8 particles on 4x4 to
8x8 periodic grids against a deliberately naive, independent evaluation:
  - gather by the direct staggered-coordinate hat-function formula (no floor logic),
  - Boris rotation by Rodrigues' formula (rotation about t by -2 atan|t|),
  - deposit via parameter-sorted crossing points (not the oracle's x-then-y split), with every
    flux / z-weight integral evaluated by Simpson's rule (exact for these polynomials),
  - curls via explicit dense difference matrices.
CPU only."""
import math

import numpy as np
import pytest

from oracle.sim import OracleSim

STAG = [(0.5, 0.0), (0.0, 0.5), (0.0, 0.0), (0.0, 0.5), (0.5, 0.0), (0.5, 0.5)]


def hat_gather(F, sx, sy, X, Y):
    ny, nx = F.shape
    val = 0.0
    for j in range(int(math.floor(Y)) - 2, int(math.floor(Y)) + 3):
        for i in range(int(math.floor(X)) - 2, int(math.floor(X)) + 3):
            w = max(0.0, 1 - abs(X - (i + sx))) * max(0.0, 1 - abs(Y - (j + sy)))
            if w > 0:
                val += w * F[j % ny, i % nx]
    return val


def rodrigues_boris(u, E, B, m_q, dt):
    h = 0.5 * dt / m_q
    um = u + h * E
    g = math.sqrt(1 + um @ um)
    t = h * B / g
    tn = np.linalg.norm(t)
    if tn > 0:
        k = t / tn
        phi = -2 * math.atan(tn)
        up = um * math.cos(phi) + np.cross(k, um) * math.sin(phi) + k * (k @ um) * (1 - math.cos(phi))
    else:
        up = um
    return up + h * E


def simpson(f, a, b):
    return (b - a) / 6 * (f(a) + 4 * f(0.5 * (a + b)) + f(b))


def naive_deposit(J, X0, Y0, Dx, Dy, q, vz, dx, dy, dt):
    ny, nx = J.shape[1:]
    ts = [0.0, 1.0]
    for (P0, D) in ((X0, Dx), (Y0, Dy)):
        if D != 0:
            lo, hi = sorted((P0, P0 + D))
            for n in range(int(math.floor(lo)) + 1, int(math.floor(hi)) + 1):
                t = (n - P0) / D
                if 0 < t < 1:
                    ts.append(t)
    ts.sort()
    for ta, tb in zip(ts[:-1], ts[1:]):
        if tb <= ta:
            continue
        tm = 0.5 * (ta + tb)
        cx, cy = int(math.floor(X0 + tm * Dx)), int(math.floor(Y0 + tm * Dy))
        a = lambda t: X0 + t * Dx - cx          # noqa: E731
        b = lambda t: Y0 + t * Dy - cy          # noqa: E731
        # charge flux through the dual faces: Jx = q dx/dt int dX (1-b) ..., Jy likewise
        J[0, cy % ny, cx % nx] += q * dx / dt * Dx * simpson(lambda t: 1 - b(t), ta, tb)
        J[0, (cy + 1) % ny, cx % nx] += q * dx / dt * Dx * simpson(b, ta, tb)
        J[1, cy % ny, cx % nx] += q * dy / dt * Dy * simpson(lambda t: 1 - a(t), ta, tb)
        J[1, cy % ny, (cx + 1) % nx] += q * dy / dt * Dy * simpson(a, ta, tb)
        for i in (0, 1):
            for j in (0, 1):
                Sx = (lambda t: 1 - a(t)) if i == 0 else a
                Sy = (lambda t: 1 - b(t)) if j == 0 else b
                J[2, (cy + j) % ny, (cx + i) % nx] += q * vz * simpson(lambda t: Sx(t) * Sy(t), ta, tb)


def diff_mats(nx, ny):
    """Dense forward / backward difference operators on the flattened (j, i) periodic grid."""
    N = nx * ny
    idx = lambda i, j: (j % ny) * nx + (i % nx)  # noqa: E731
    Dxf, Dxb, Dyf, Dyb = (np.zeros((N, N)) for _ in range(4))
    for j in range(ny):
        for i in range(nx):
            r = idx(i, j)
            Dxf[r, idx(i + 1, j)] += 1; Dxf[r, r] -= 1
            Dxb[r, r] += 1; Dxb[r, idx(i - 1, j)] -= 1
            Dyf[r, idx(i, j + 1)] += 1; Dyf[r, r] -= 1
            Dyb[r, r] += 1; Dyb[r, idx(i, j - 1)] -= 1
    return Dxf, Dxb, Dyf, Dyb


def naive_yee(E, B, J, dx, dy, dt):
    ny, nx = E.shape[1:]
    Dxf, Dxb, Dyf, Dyb = diff_mats(nx, ny)
    e = [E[c].ravel().copy() for c in range(3)]
    b = [B[c].ravel().copy() for c in range(3)]
    j = [J[c].ravel() for c in range(3)]

    def bhalf():
        b[0] -= 0.5 * dt * (Dyf @ e[2]) / dy
        b[1] += 0.5 * dt * (Dxf @ e[2]) / dx
        b[2] += 0.5 * dt * ((Dyf @ e[0]) / dy - (Dxf @ e[1]) / dx)
    bhalf()
    e[0] += dt * ((Dyb @ b[2]) / dy - j[0])
    e[1] += dt * (-(Dxb @ b[2]) / dx - j[1])
    e[2] += dt * ((Dxb @ b[1]) / dx - (Dyb @ b[0]) / dy - j[2])
    bhalf()
    return np.stack([v.reshape(ny, nx) for v in e]), np.stack([v.reshape(ny, nx) for v in b])


def make_case(seed, nx, ny, npart):
    rng = np.random.default_rng(seed)
    ix = rng.integers(0, nx, npart).astype(np.int32)
    iy = rng.integers(0, ny, npart).astype(np.int32)
    x, y = rng.random(npart), rng.random(npart)
    u = rng.normal(size=(3, npart)) * 2.0
    if npart >= 4:
        x[0] = 0.0                                   # exactly on an edge
        y[1] = 0.0
        x[2], y[2], u[0, 2], u[1, 2] = 0.9, 0.9, 3.0, 3.0    # corner / double crossing
        x[3], y[3], u[0, 3], u[1, 3] = 0.05, 0.95, -3.0, 3.0
    E = rng.normal(size=(3, ny, nx))
    B = rng.normal(size=(3, ny, nx))
    return ix, iy, x, y, u, E, B


@pytest.mark.parametrize("seed,nx,ny,npart", [(1, 4, 4, 1), (2, 5, 4, 3), (3, 6, 6, 8), (4, 8, 5, 8), (5, 7, 8, 6)])
def test_one_step_bruteforce(seed, nx, ny, npart):
    dx, dy, dt, m_q = 0.1, 0.12, 0.07, -1.0
    ix, iy, x, y, u, E, B = make_case(seed, nx, ny, npart)
    sp = [dict(m_q=m_q, n=1.0, ppc=(2, 2), ufl=(0, 0, 0), uth=(0, 0, 0), ix=ix, iy=iy, x=x, y=y,
               ux=u[0], uy=u[1], uz=u[2])]
    sim = OracleSim(nx, ny, dx, dy, dt, sp, E=E, B=B)
    q = -1.0 / 4
    sim.step()
    # naive
    J = np.zeros((3, ny, nx))
    X1 = np.zeros(npart); Y1 = np.zeros(npart); U1 = np.zeros((3, npart))
    for p in range(npart):
        X, Y = ix[p] + x[p], iy[p] + y[p]
        Ep = np.array([hat_gather(E[c], *STAG[c], X, Y) for c in range(3)])
        Bp = np.array([hat_gather(B[c], *STAG[3 + c], X, Y) for c in range(3)])
        un = rodrigues_boris(u[:, p].copy(), Ep, Bp, m_q, dt)
        g = math.sqrt(1 + un @ un)
        Dx, Dy = un[0] / g * dt / dx, un[1] / g * dt / dy
        naive_deposit(J, X, Y, Dx, Dy, q, un[2] / g, dx, dy, dt)
        X1[p], Y1[p], U1[:, p] = X + Dx, Y + Dy, un
    En, Bn = naive_yee(E, B, J, dx, dy, dt)
    s = sim.species[0]
    assert np.allclose(np.stack([s["ux"], s["uy"], s["uz"]]), U1, atol=1e-13, rtol=1e-13)
    Xo = s["ix"] + s["x"]
    Yo = s["iy"] + s["y"]
    assert np.allclose(Xo, np.mod(X1, nx), atol=1e-13)
    assert np.allclose(Yo, np.mod(Y1, ny), atol=1e-13)
    assert np.all((s["x"] >= 0) & (s["x"] < 1) & (s["y"] >= 0) & (s["y"] < 1))
    assert np.allclose(sim.fields(2), J, atol=1e-13)
    assert np.allclose(sim.fields(0), En, atol=1e-12)
    assert np.allclose(sim.fields(1), Bn, atol=1e-12)
