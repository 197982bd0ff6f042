"""The five workloads of BASELINE.json (configs[0..4] = C1..C5) as plain dicts.

Readings of what BASELINE.json leaves open are SURVEY.md §8(c): seeds R10, C3's 8 ppc as
(4, 2) R11, C4 filter passes R12, C4 laser R17, C4 ramp R16.  Boundary codes follow
include/zpic.h: 0 periodic, 1 open (removal + Mur-1), 2 moving window (x only).
"""
import copy

PERIODIC, OPEN, WINDOW = 0, 1, 2


def _electrons(n, ppc, ufl=(0.0, 0.0, 0.0), uth=(0.0, 0.0, 0.0), profile="uniform", x0=0.0, x1=0.0, m_q=-1.0):
    return {"m_q": float(m_q), "ppc": tuple(ppc), "n": float(n), "ufl": tuple(float(v) for v in ufl),
            "uth": tuple(float(v) for v in uth), "profile": profile, "x0": float(x0), "x1": float(x1)}


CONFIGS = {
    # BASELINE.json configs[0]: uniform thermal plasma 64x64, 4x4 ppc, uth 0.1, 100 steps
    "C1": {"name": "C1-uniform-64", "nx": 64, "ny": 64, "dx": 0.1, "dy": 0.1, "dt": 0.07,
           "bc": (PERIODIC, PERIODIC), "steps": 100, "seed": 101,
           "species": [_electrons(1.0, (4, 4), uth=(0.1, 0.1, 0.1))]},
    # configs[1]: counter-streaming (Weibel) 256^2, two electron species, uz = +-0.6, 500 steps
    "C2": {"name": "C2-weibel-256", "nx": 256, "ny": 256, "dx": 0.1, "dy": 0.1, "dt": 0.07,
           "bc": (PERIODIC, PERIODIC), "steps": 500, "seed": 202,
           "species": [_electrons(0.5, (4, 4), ufl=(0, 0, 0.6), uth=(0.05, 0.05, 0.05)),
                       _electrons(0.5, (4, 4), ufl=(0, 0, -0.6), uth=(0.05, 0.05, 0.05))]},
    # configs[2]: collision of plasma clouds 2048x1024, open x, periodic y, 8 ppc (4,2), 1000 steps
    "C3": {"name": "C3-clouds-2048x1024", "nx": 2048, "ny": 1024, "dx": 0.1, "dy": 0.1, "dt": 0.07,
           "bc": (OPEN, PERIODIC), "steps": 1000, "seed": 303,
           "species": [_electrons(1.0, (4, 2), ufl=(0.5, 0, 0), uth=(0.02, 0.02, 0.02), profile="slab",
                                  x0=0.0, x1=102.4),
                       _electrons(1.0, (4, 2), ufl=(-0.5, 0, 0), uth=(0.02, 0.02, 0.02), profile="slab",
                                  x0=102.4, x1=204.8)]},
    # configs[3]: LWFA 4000x512, dx 0.02, dy 0.1, dt 0.019, moving window, ramp at x=20 over 20 cells
    "C4": {"name": "C4-lwfa-4000x512", "nx": 4000, "ny": 512, "dx": 0.02, "dy": 0.1, "dt": 0.019,
           "bc": (WINDOW, OPEN), "steps": 4000, "seed": 404,
           "species": [_electrons(1.0, (2, 2), profile="ramp", x0=20.0, x1=20.0 + 20 * 0.02)],
           "filter": (4, 1),
           "laser": {"a0": 2.0, "omega0": 10.0, "fwhm": 2.0, "W0": 4.0, "start": 78.0, "polarization": "y"}},
    # configs[4]: large uniform thermal plasma 8192^2, 4x4 ppc (1.07e9 particles), 50 steps
    "C5": {"name": "C5-uniform-8192", "nx": 8192, "ny": 8192, "dx": 0.1, "dy": 0.1, "dt": 0.07,
           "bc": (PERIODIC, PERIODIC), "steps": 50, "seed": 505,
           "species": [_electrons(1.0, (4, 4), uth=(0.1, 0.1, 0.1))]},
    # ---- the paper's own workloads, B200-sized --------
    # Readings: the paper gives grid, ppc, species and step counts only; dx, dy,
    # dt, densities, drifts and temperatures reuse C2's (Weibel) and C4's (LWFA) values.
    # Weibel: electron + positron clouds moving along +-z, 512^2, 256 ppc each
    # (16 x 16), 500 steps -> 134,217,728 particles.
    "P-WEIBEL": {"name": "paper-weibel-pairs-512", "nx": 512, "ny": 512, "dx": 0.1, "dy": 0.1, "dt": 0.07,
                 "bc": (PERIODIC, PERIODIC), "steps": 500, "seed": 606,
                 "species": [_electrons(0.5, (16, 16), ufl=(0, 0, 0.6), uth=(0.05, 0.05, 0.05)),
                             _electrons(0.5, (16, 16), ufl=(0, 0, -0.6), uth=(0.05, 0.05, 0.05), m_q=1.0)]},
    # LWFA: 2000 x 512 cells, 16 ppc (4 x 4), 4000 steps, moving window,
    # compensated filter; C4's dx, dy, dt, laser and ramp with the laser's leading edge at Lx - 2.
    "P-LWFA": {"name": "paper-lwfa-2000x512", "nx": 2000, "ny": 512, "dx": 0.02, "dy": 0.1, "dt": 0.019,
               "bc": (WINDOW, OPEN), "steps": 4000, "seed": 707,
               "species": [_electrons(1.0, (4, 4), profile="ramp", x0=20.0, x1=20.0 + 20 * 0.02)],
               "filter": (4, 1),
               "laser": {"a0": 2.0, "omega0": 10.0, "fwhm": 2.0, "W0": 4.0, "start": 38.0, "polarization": "y"}},
    # Uniform cold / warm plasmas of the weak-scaling test: 16 x 16 ppc,
    # u_th = 0 / 0.01; the grid per GPU is fixed (1024^2 here) and the global grid grows with N.
    "P-COLD": {"name": "paper-uniform-cold", "nx": 1024, "ny": 1024, "dx": 0.1, "dy": 0.1, "dt": 0.07,
               "bc": (PERIODIC, PERIODIC), "steps": 500, "seed": 808,
               "species": [_electrons(1.0, (16, 16))]},
    "P-WARM": {"name": "paper-uniform-warm", "nx": 1024, "ny": 1024, "dx": 0.1, "dy": 0.1, "dt": 0.07,
               "bc": (PERIODIC, PERIODIC), "steps": 500, "seed": 909,
               "species": [_electrons(1.0, (16, 16), uth=(0.01, 0.01, 0.01))]},
}


def config(name, **overrides):
    """A deep copy of a named config with top-level keys overridden (e.g. nx=, ny=, steps=)."""
    c = copy.deepcopy(CONFIGS[name])
    c.update(overrides)
    return c


def charge(sp):
    """Per-particle charge q_s = sign(m_q) * n_s / (ppc_x * ppc_y).
    A normalisation of the initial condition, shared as an input by both sides."""
    sign = 1.0 if sp["m_q"] > 0 else -1.0
    return sign * sp["n"] / (sp["ppc"][0] * sp["ppc"][1])
