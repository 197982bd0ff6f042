"""Seeded initial-condition generators (numpy, fp64 -> fp32).

RNG: a counter-based generator, so every particle's
momentum depends only on (seed, species index, particle id) and not on the decomposition.
    mix64(z): z += 0x9E3779B97F4A7C15; z = (z ^ z>>30) * 0xBF58476D1CE4E5B9;
              z = (z ^ z>>27) * 0x94D049BB133111EB; return z ^ z>>31       (splitmix64)
    key      = mix64(mix64(seed) + species)
    r(id, j) = mix64(key ^ mix64(8*id + j)),   j = 0..5
    U_j      = ((r >> 11) + 0.5) * 2^-53                                  in (0, 1)
    N_k      = sqrt(-2 ln U_{2k}) * cos(2 pi U_{2k+1}),  k = 0, 1, 2       (Box-Muller)
    u_k      = fp32(ufl_k + uth_k * N_k)       (fp64 multiply, then fp64 add, then round)
The CUDA injector implements the same generator independently (K0 `k_inject` in
paper_2106_12485_b200/csrc/zpic_kernels.cu).

Particle ids (SURVEY.md §8(c) "Initial state"): the global sub-lattice index
    id = ((iy * nx + ix) * ppc_y + l) * ppc_x + k
for sub-lattice point (k, l) of cell (ix, iy), x = (k + 1/2)/ppc_x, y = (l + 1/2)/ppc_y.
"""
import math

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_G = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def mix64(z):
    """splitmix64 finaliser on uint64 arrays (wrap-around arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + _G
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def uniforms(seed, species, ids, j):
    """U_j(id) in (0,1), fp64."""
    key = mix64(mix64(np.uint64(seed)) + np.uint64(species))
    with np.errstate(over="ignore"):
        ctr = np.asarray(ids, dtype=np.uint64) * np.uint64(8) + np.uint64(j)
    r = mix64(key ^ mix64(ctr))
    return ((r >> np.uint64(11)).astype(np.float64) + 0.5) * (2.0 ** -53)


def normals(seed, species, ids):
    """(3, n) fp64 standard normals N_0, N_1, N_2 per particle id."""
    out = np.empty((3, len(ids)), dtype=np.float64)
    for k in range(3):
        u1 = uniforms(seed, species, ids, 2 * k)
        u2 = uniforms(seed, species, ids, 2 * k + 1)
        out[k] = np.sqrt(-2.0 * np.log(u1)) * np.cos(6.283185307179586 * u2)
    return out


def momenta(sp, seed, species, ids):
    """u = ufl + uth * N, computed in fp64 (multiply then add), rounded to fp32."""
    n = normals(seed, species, ids) if any(v != 0.0 for v in sp["uth"]) else np.zeros((3, len(ids)))
    u = []
    for k in range(3):
        u.append((np.float64(sp["ufl"][k]) + np.float64(sp["uth"][k]) * n[k]).astype(np.float32))
    return u


def lattice_species(nx, ny, ppc, cell_mask=None):
    """Regular ppc sub-lattice in every cell with cell_mask[iy, ix] True (all cells if None).
    Returns ix, iy (int32), x, y (fp32), id (uint64) sorted by id."""
    px, py = ppc
    if cell_mask is None:
        cy, cx = np.divmod(np.arange(nx * ny, dtype=np.int64), nx)
    else:
        cy, cx = np.nonzero(cell_mask)
        cy = cy.astype(np.int64)
        cx = cx.astype(np.int64)
    l, k = np.divmod(np.arange(px * py, dtype=np.int64), px)
    ix = np.repeat(cx, px * py)
    iy = np.repeat(cy, px * py)
    kk = np.tile(k, len(cx))
    ll = np.tile(l, len(cx))
    ids = ((iy * nx + ix) * py + ll) * px + kk
    x = ((kk + 0.5) / px).astype(np.float32)
    y = ((ll + 0.5) / py).astype(np.float32)
    return ix.astype(np.int32), iy.astype(np.int32), x, y, ids.astype(np.uint64)


def species_particles(cfg, s):
    """Particles of species s of config cfg as a dict of numpy arrays (ix, iy, x, y, ux, uy,
    uz, id).  Profiles: 'uniform'; 'slab' (cell centre x in [x0, x1)); 'ramp' (R16)."""
    sp = cfg["species"][s]
    nx, ny = cfg["nx"], cfg["ny"]
    if sp["profile"] == "ramp":
        return ramp_species(cfg, s)
    mask = None
    if sp["profile"] == "slab":
        xc = (np.arange(nx) + 0.5) * cfg["dx"]
        colmask = (xc >= sp["x0"]) & (xc < sp["x1"])
        mask = np.broadcast_to(colmask[None, :], (ny, nx))
    ix, iy, x, y, ids = lattice_species(nx, ny, sp["ppc"], mask)
    ux, uy, uz = momenta(sp, cfg["seed"], s, ids)
    return {"ix": ix, "iy": iy, "x": x, "y": y, "ux": ux, "uy": uy, "uz": uz,
            "id": ids.astype(np.uint32)}


def patch_species(cfg, s, gx0, gy0, w, h):
    """The particles of the uniform species s whose cells lie in the w x h patch with global
    origin (gx0, gy0) (periodic wrap of the global grid), with their GLOBAL ids and momenta, and
    cell indices relative to the patch.  Used to rebuild a sub-domain of a full-size workload
    exactly as the full lattice has it (the full-size sampled parity checks)."""
    sp = cfg["species"][s]
    nx, ny = cfg["nx"], cfg["ny"]
    px, py = sp["ppc"]
    lx, ly = np.meshgrid(np.arange(w), np.arange(h))
    lx, ly = lx.ravel(), ly.ravel()
    gx, gy = (gx0 + lx) % nx, (gy0 + ly) % ny
    l, k = np.divmod(np.arange(px * py, dtype=np.int64), px)
    rep = px * py
    ids = ((np.repeat(gy, rep).astype(np.int64) * nx + np.repeat(gx, rep)) * py + np.tile(l, len(gx))) * px + np.tile(k, len(gx))
    ux, uy, uz = momenta(sp, cfg["seed"], s, ids.astype(np.uint64))
    return {"ix": np.repeat(lx, rep).astype(np.int32), "iy": np.repeat(ly, rep).astype(np.int32),
            "x": ((np.tile(k, len(gx)) + 0.5) / px).astype(np.float32),
            "y": ((np.tile(l, len(gx)) + 0.5) / py).astype(np.float32),
            "ux": ux, "uy": uy, "uz": uz, "id": ids.astype(np.uint32)}


def ramp_species(cfg, s):
    """C4 density (R16): n = 0 for x < x0, linear 0 -> n over [x0, x1), n beyond; equal-charge
    particles.  Along x, every y sub-lattice row places particles by inverting the cumulative
    density: in the ramp X_k = x0 + sqrt(2 L (k + 1/2) dx / ppc_x), L = x1 - x0,
    k < ppc_x L / (2 dx); from x1 on, the regular sub-lattice.  ids: the row-major order of the
    resulting list (row of cells iy, then sub-row l, then x)."""
    sp = cfg["species"][s]
    nx, ny, dx = cfg["nx"], cfg["ny"], cfg["dx"]
    px, py = sp["ppc"]
    x0, x1 = sp["x0"], sp["x1"]
    L = x1 - x0
    nramp = int(round(px * L / (2.0 * dx)))
    k = np.arange(nramp, dtype=np.float64)
    Xr = x0 + np.sqrt(2.0 * L * (k + 0.5) * dx / px)
    first = int(math.ceil(x1 / dx - 1e-9))
    cols = np.arange(first, nx, dtype=np.float64)
    Xu = ((cols[:, None] + (np.arange(px)[None, :] + 0.5) / px) * dx).ravel()
    X = np.concatenate([Xr, Xu])            # one x sub-row of particles (physical x)
    gx = X / dx
    ixr = np.floor(gx).astype(np.int64)
    xr = (gx - ixr).astype(np.float32)
    up = xr >= np.float32(1.0)          # an offset that rounds to 1 in fp32 starts the next cell (R6)
    ixr[up] += 1
    xr[up] = 0.0
    n_row = len(X)
    rows = np.arange(ny * py, dtype=np.int64)          # y sub-rows: iy = r // py, l = r % py
    iy = np.repeat(rows // py, n_row)
    yy = np.repeat(((rows % py) + 0.5) / py, n_row)
    ix = np.tile(ixr, ny * py)
    x = np.tile(xr, ny * py)
    ids = np.arange(len(ix), dtype=np.uint64)
    ux, uy, uz = momenta(sp, cfg["seed"], s, ids)
    return {"ix": ix.astype(np.int32), "iy": iy.astype(np.int32), "x": x.astype(np.float32),
            "y": yy.astype(np.float32), "ux": ux, "uy": uy, "uz": uz, "id": ids.astype(np.uint32)}


def laser_fields(cfg):
    """C4 laser (R17): E_y = a0 w0 env(x) exp(-(y - yc)^2 / W0^2) cos(w0 (x - xc)) and B_z = E_y
    at B_z's staggered points (+x propagation); env = sin^2 hump of total length 2 fwhm whose
    leading edge is at x = start (field FWHM = fwhm); xc = start - fwhm; yc = Ly / 2.
    Returns E, B as fp32 arrays (3, ny, nx) [comp][y][x] (interior values)."""
    las = cfg["laser"]
    nx, ny, dx, dy = cfg["nx"], cfg["ny"], cfg["dx"], cfg["dy"]
    a0, w0, fwhm, W0, start = las["a0"], las["omega0"], las["fwhm"], las["W0"], las["start"]
    xc, yc = start - fwhm, 0.5 * ny * dy
    lo = start - 2.0 * fwhm

    def prof(xp, yp):
        env = np.where((xp >= lo) & (xp <= start), np.sin(np.pi * (xp - lo) / (2.0 * fwhm)) ** 2, 0.0)
        return a0 * w0 * env * np.exp(-((yp - yc) ** 2) / W0 ** 2) * np.cos(w0 * (xp - xc))

    i = np.arange(nx, dtype=np.float64)
    j = np.arange(ny, dtype=np.float64)
    E = np.zeros((3, ny, nx), dtype=np.float32)
    B = np.zeros((3, ny, nx), dtype=np.float32)
    E[1] = prof((i[None, :]) * dx, (j[:, None] + 0.5) * dy)          # Ey at (i, j+1/2)
    B[2] = prof((i[None, :] + 0.5) * dx, (j[:, None] + 0.5) * dy)    # Bz at (i+1/2, j+1/2)
    return E, B
