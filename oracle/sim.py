"""The oracle's time step, in the order of SURVEY.md §8(c) "Step n -> n+1" (PAPER.md:142-146,
Fig. 1).  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  The loops are in
oracle/zpic_oracle.c; this file only sequences them and does the particle bookkeeping
(boundaries, moving window) with plain numpy.

State at the start of step n: E^n, B^n (fp64, guard-extended, guards valid), particles
(ix, iy, x, y) at t_n and u^{n-1/2} (fp64).
"""
import numpy as np

from . import lib

PERIODIC, OPEN, WINDOW = 0, 1, 2


class OracleSim:
    def __init__(self, nx, ny, dx, dy, dt, species, bc=(PERIODIC, PERIODIC), filter_=(0, 0),
                 E=None, B=None, seed=0):
        """species: list of dicts with m_q, n, ppc, ufl, uth and the particle arrays ix, iy,
        x, y, ux, uy, uz (any dtype; promoted to int32 / fp64) and optional id.
        E, B: optional interior initial fields, arrays (3, ny, nx)."""
        self.nx, self.ny, self.dx, self.dy, self.dt = nx, ny, dx, dy, dt
        self.bcx, self.bcy = bc
        self.filter = filter_
        self.seed = seed
        self.E = lib.grid(nx, ny)
        self.B = lib.grid(nx, ny)
        self.J = lib.grid(nx, ny)
        self.J_prefilter = lib.grid(nx, ny)
        if E is not None:
            self.E[:, 1:ny + 1, 1:nx + 1] = np.asarray(E, dtype=np.float64)
        if B is not None:
            self.B[:, 1:ny + 1, 1:nx + 1] = np.asarray(B, dtype=np.float64)
        lib.refresh_guards(self.E, self.bcx, self.bcy, True)
        lib.refresh_guards(self.B, self.bcx, self.bcy, False)
        self.species = []
        for sp in species:
            s = {k: sp[k] for k in ("m_q", "n", "ppc", "ufl", "uth")}
            s.update({k: sp[k] for k in ("profile", "x0", "x1") if k in sp})
            # per-particle charge q_s = sign(m_q) n_s / (ppc_x ppc_y)  (R8)
            s["q"] = (1.0 if sp["m_q"] > 0 else -1.0) * sp["n"] / (sp["ppc"][0] * sp["ppc"][1])
            for k in ("ix", "iy"):
                s[k] = np.ascontiguousarray(sp[k], dtype=np.int32).copy()
            for k in ("x", "y", "ux", "uy", "uz"):
                s[k] = np.ascontiguousarray(sp[k], dtype=np.float64).copy()
            s["id"] = np.asarray(sp["id"]).astype(np.int64).copy() if "id" in sp else np.arange(len(s["ix"]))
            self.species.append(s)
        self.n = 0            # time level of the state
        self.n_move = 0       # moving-window shifts so far
        self.fe = []          # FE(n), n = 0 .. steps-1
        self.ke = []          # [KE_s(n)]
        self.bad_moves = 0

    # ---------------------------------------------------------------------------------
    def step(self):
        nx, ny, dx, dy, dt = self.nx, self.ny, self.dx, self.dy, self.dt
        # 1. J <- 0, including guards
        self.J[...] = 0.0
        ke = []
        # 2. every particle: interpolate (A1) -> Boris (A2) -> deposit + cell update (A3)
        for s in self.species:
            Ep, Bp = lib.interpolate(self.E, self.B, s["ix"], s["iy"], s["x"], s["y"])
            k = lib.boris(s["ux"], s["uy"], s["uz"], Ep, Bp, s["m_q"], dt)
            ke.append(s["q"] * s["m_q"] * dx * dy * k)
            self.bad_moves += lib.advance_deposit(s["ix"], s["iy"], s["x"], s["y"], s["ux"], s["uy"], s["uz"],
                                                  s["q"], dt, dx, dy, self.J)
        # 3. particle boundaries (a5): periodic wrap, or removal on an open axis.  A moving-window
        #    x axis is handled after the window shift (step 7).
        for s in self.species:
            self._particle_bc(s, window_now=False)
        # 4. ghost-current reduction (a7)
        lib.fold_current(self.J, self.bcx, self.bcy)
        self.J_prefilter[...] = self.J
        # 5. filter (a8)
        if self.filter[0] > 0:
            lib.filter_x(self.J, self.bcx, self.bcy, self.filter[0], self.filter[1])
        # 6. FE(n) on the inputs, then the Yee advance (a9, a10)
        self.fe.append(lib.field_energy(self.E, self.B, dx, dy))
        lib.yee_advance(self.E, self.B, self.J, dt, dx, dy, self.bcx, self.bcy)
        self.ke.append(ke)
        # 7. n <- n+1; moving window (a11)
        self.n += 1
        if self.bcx == WINDOW:
            if self.n * dt > dx * (self.n_move + 1):
                self._shift_window()
            for s in self.species:
                self._particle_bc(s, window_now=True)

    def run(self, n):
        for _ in range(n):
            self.step()

    # ---------------------------------------------------------------------------------
    def _keep(self, s, m):
        if m.all():    # nothing removed (bookkeeping only: skip the copies)
            return
        for k in ("ix", "iy", "x", "y", "ux", "uy", "uz", "id"):
            s[k] = np.ascontiguousarray(s[k][m])

    def _particle_bc(self, s, window_now):
        nx, ny = self.nx, self.ny
        if not window_now:
            if self.bcx == PERIODIC:
                s["ix"] = np.ascontiguousarray(np.mod(s["ix"], nx).astype(np.int32))
            elif self.bcx == OPEN:
                self._keep(s, (s["ix"] >= 0) & (s["ix"] < nx))
            if self.bcy == PERIODIC:
                s["iy"] = np.ascontiguousarray(np.mod(s["iy"], ny).astype(np.int32))
            elif self.bcy == OPEN:
                self._keep(s, (s["iy"] >= 0) & (s["iy"] < ny))
        else:
            self._keep(s, (s["ix"] >= 0) & (s["ix"] < nx))

    def _shift_window(self):
        """Shift E, B one column toward -x (new column nx-1 is zero); every particle ix -= 1;
        inject a fresh column at ix = nx-1 (R14, R15).  Particles with ix < 0 are removed by the
        caller."""
        nx, ny = self.nx, self.ny
        for F in (self.E, self.B):
            F[:, :, 1:nx] = F[:, :, 2:nx + 1]
            F[:, :, nx] = 0.0
            lib.refresh_guards(F, self.bcx, self.bcy, F is self.E)
        for si, s in enumerate(self.species):
            s["ix"] -= 1
            inj = self._inject_column(si, s)
            if inj is not None:
                for k in ("ix", "iy", "x", "y", "ux", "uy", "uz", "id"):
                    s[k] = np.ascontiguousarray(np.concatenate([s[k], inj[k].astype(s[k].dtype)]))
        self.n_move += 1

    def _inject_column(self, si, s):
        """Fresh plasma in column nx-1 (R15): density = the species profile at the column's
        absolute position x = (nx - 1 + n_move + 1) dx, i.e. beyond the initial box.  Readings
        (DESIGN.md §2): a uniform profile gives n there; a ramp that ends inside the initial box
        (x1 <= nx dx: C4, P-LWFA) gives n for every injected column; a slab profile, or a ramp
        reaching past the box, is not a supported moving-window input (the library rejects it at
        zpic_init).  Density n > 0 -> the ppc sub-lattice; n = 0 -> nothing.  Momenta from the
        shared seeded generator (synth), keyed by id = 2^31 + (n_move*ny + iy)*ppc + l*ppc_x + k."""
        from synth.generate import momenta
        nx, ny = self.nx, self.ny
        prof = s.get("profile", "uniform")
        if prof == "slab" or (prof == "ramp" and s["x1"] > nx * self.dx):
            raise ValueError("moving-window injection needs a uniform profile or a ramp inside the box (R15)")
        if not s["n"] > 0:
            return None
        px, py = s["ppc"]
        l, k = np.divmod(np.arange(px * py), px)
        iy = np.repeat(np.arange(ny), px * py)
        ll = np.tile(l, ny)
        kk = np.tile(k, ny)
        ids = (2 ** 31 + (self.n_move * ny + iy) * px * py + ll * px + kk).astype(np.uint64)
        ux, uy, uz = momenta(s, self.seed, si, ids)
        return {"ix": np.full(len(iy), nx - 1, np.int32), "iy": iy.astype(np.int32),
                "x": (kk + 0.5) / px, "y": (ll + 0.5) / py,
                "ux": ux.astype(np.float64), "uy": uy.astype(np.float64), "uz": uz.astype(np.float64),
                "id": ids.astype(np.int64)}

    # ---------------------------------------------------------------------------------
    def fields(self, which):
        """Interior [comp][y][x] of E (0), B (1), J (2, after fold + filter), J pre-filter (3)."""
        F = (self.E, self.B, self.J, self.J_prefilter)[which]
        return F[:, 1:self.ny + 1, 1:self.nx + 1].copy()


def from_config(cfg, particles=None, E=None, B=None):
    """An OracleSim for a synth config; particles: list (per species) of dicts of arrays."""
    from synth.generate import species_particles, laser_fields
    if particles is None:
        particles = [species_particles(cfg, s) for s in range(len(cfg["species"]))]
    if E is None and B is None and cfg.get("laser"):
        E, B = laser_fields(cfg)
    sp = []
    for s, p in zip(cfg["species"], particles):
        d = dict(s)
        d.update(p)
        sp.append(d)
    return OracleSim(cfg["nx"], cfg["ny"], cfg["dx"], cfg["dy"], cfg["dt"], sp, bc=tuple(cfg["bc"]),
                     filter_=tuple(cfg.get("filter", (0, 0))), E=E, B=B, seed=cfg["seed"])
