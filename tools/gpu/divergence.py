"""How fast two GPU runs of the same config drift apart when only the rounding differs: the
one-word vs the exact two-word tile current (both within the north-star bars at step 10), and a
1-ulp change of one particle's x.  Prints the relative L2 distance of E and B between the runs
every `every` steps (unstable physics amplifies any rounding difference: the final-map comparison
of PAPER.md:351-353 is meaningful only while that growth stays small).
usage: python tools/gpu/divergence.py CONFIG STEPS EVERY"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import fullrun_specs as F  # noqa: E402
import paper_2106_12485_b200 as z  # noqa: E402

name, steps, every = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])


def run(precision, perturb=False):
    cfg, parts, E, B = F.inputs(name)
    g = z.Simulation(cfg, inject=False, current_precision=precision)
    for s, p in enumerate(parts):
        if perturb and s == 0:
            p = {k: v.copy() for k, v in p.items()}
            p["x"][0] = np.nextafter(p["x"][0], np.float32(1.0))
        g.set_particles(s, p)
    if E is not None:
        g.set_fields(0, E)
        g.set_fields(1, B)
    out = {}
    for n in range(1, steps + 1):
        g.step(1)
        if n % every == 0 or n in (1, 10):
            out[n] = (g.fields(0).astype(np.float64), g.fields(1).astype(np.float64))
    g.close()
    return out


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


a = run("auto")
b = run("exact")
c = run("auto", perturb=True)
for n in sorted(a):
    print(json.dumps({"config": name, "step": n,
                      "auto_vs_exact": {"E": rel(a[n][0], b[n][0]), "B": rel(a[n][1], b[n][1])},
                      "auto_vs_1ulp": {"E": rel(a[n][0], c[n][0]), "B": rel(a[n][1], c[n][1])}}), flush=True)
