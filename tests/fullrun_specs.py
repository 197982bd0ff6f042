"""The full-length parity runs (BASELINE.json north_star: "over the full run, the discrete
continuity residual must stay <= 1e-5 and the field and kinetic energy histories must agree to
within 1 %"; PAPER.md:351-353 compares the final magnetic-field map).  One definition of each run,
shared by the background oracle jobs (tests/oracle_job.py, started by tests/conftest.py so the
long fp64 runs overlap the GPU tests) and by the GPU side (tests/test_fullrun_gpu.py).  Both sides
start from the same synth arrays.  CPU-only; imports neither side's arithmetic."""
import synth

# name -> (BASELINE config, steps, steps whose interior E, B the oracle job saves)
RUNS = {
    "C1": ("C1", 100, (10, 100)),     # configs[0], its whole run
    "C2": ("C2", 500, (10, 500)),     # configs[1], its whole run (Weibel growth and saturation)
    "C3": ("C3", 200, (10, 200)),     # configs[2], full grid, the first 200 of 1000 steps
    "C4": ("C4", 200, (10, 200)),     # configs[3], full grid, the first 200 of 4000 steps
    # their whole runs (oracle ~30 / > 46 min, C4 beyond a 60-min gpurun call beside C3: only with
    # ZPIC_FULLRUN_LONG=1, test_fullrun_gpu.py)
    "C3-whole": ("C3", 1000, (10, 1000)),
    "C4-whole": ("C4", 4000, (10, 4000)),
}

# C5 (configs[4], 1.07e9 particles) is checked on periodic patches of the global lattice: after k
# steps the patch interior beyond a margin of 2k + 4 cells is exactly the full-domain evolution
# (a step's stencils reach 2 cells).  Patch origins: interior, both periodic seams, tile corners.
C5_STEPS = 50
C5_PATCH = 256
C5_MARGIN = 2 * C5_STEPS + 4
C5_ORIGINS = ((1000, 3000), (8192 - 130, 8192 - 120), (4090 - 100, 6140 - 100))
C5_SNAPS = (1, 10, 25, 50)


def config(name):
    return synth.config(RUNS[name][0])


def inputs(name):
    """(cfg, per-species particle dicts, initial E, initial B): the shared seeded inputs."""
    cfg = config(name)
    parts = [synth.species_particles(cfg, s) for s in range(len(cfg["species"]))]
    E = B = None
    if cfg.get("laser"):
        E, B = synth.laser_fields(cfg)
    return cfg, parts, E, B


def c5_patch(cfg, origin):
    """The species dict + particles of the C5 patch at a global origin (synth.patch_species)."""
    p = synth.generate.patch_species(cfg, 0, origin[0], origin[1], C5_PATCH, C5_PATCH)
    sp = dict(cfg["species"][0])
    sp.update(p)
    return sp
