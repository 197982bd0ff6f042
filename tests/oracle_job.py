"""One long oracle run in its own process (TEST INFRASTRUCTURE ONLY: started by tests/conftest.py
for tests/test_fullrun_gpu.py, so the serial fp64 runs overlap the GPU tests on the host's other
cores).  Usage: python tests/oracle_job.py NAME OUT.npz

Writes fe[n], ke[n, s] for n = 0 .. steps-1 (the oracle's FE(n), KE_s(n))
and the interior E, B after each snapshot step; for C5, the patch fields at the snapshot steps."""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import fullrun_specs as F  # noqa: E402
from oracle.sim import OracleSim, from_config  # noqa: E402


def run_config(name, out):
    cfg, parts, E, B = F.inputs(name)
    _, steps, snaps = F.RUNS[name]
    o = from_config(cfg, particles=parts, E=E, B=B)
    res = {}
    t0 = time.time()
    for n in range(1, steps + 1):
        o.step()
        if n in snaps:
            res["E%d" % n] = o.fields(0)
            res["B%d" % n] = o.fields(1)
    res["fe"] = np.array(o.fe)
    res["ke"] = np.array(o.ke)
    res["particles"] = np.array([len(s["ix"]) for s in o.species])
    res["seconds"] = np.array(time.time() - t0)
    np.savez(out + ".tmp.npz", **res)
    os.replace(out + ".tmp.npz", out)


def run_c5(out):
    import synth
    cfg = synth.config("C5")
    res = {}
    t0 = time.time()
    for k, origin in enumerate(F.C5_ORIGINS):
        sp = F.c5_patch(cfg, origin)
        o = OracleSim(F.C5_PATCH, F.C5_PATCH, cfg["dx"], cfg["dy"], cfg["dt"], [sp])
        for n in range(1, F.C5_STEPS + 1):
            o.step()
            if n in F.C5_SNAPS:
                res["p%d_E%d" % (k, n)] = o.fields(0)
                res["p%d_B%d" % (k, n)] = o.fields(1)
    res["seconds"] = np.array(time.time() - t0)
    np.savez(out + ".tmp.npz", **res)
    os.replace(out + ".tmp.npz", out)


if __name__ == "__main__":
    name, out = sys.argv[1], sys.argv[2]
    if name == "C5":
        run_c5(out)
    else:
        run_config(name, out)
