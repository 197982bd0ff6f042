"""Same-box bit-identity check of two library variants: run a config for N steps with the
library named by ZPIC_SO and write E, B, J and the energy history to OUT.npz; compare two
outputs with --compare A.npz B.npz.  usage: python tools/gpu/bitcmp.py CONFIG STEPS OUT.npz"""
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))

if sys.argv[1] == "--compare":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    bad = [k for k in a.files if not np.array_equal(a[k], b[k])]
    for k in bad:
        d = np.abs(a[k].astype(np.float64) - b[k]).max()
        print("DIFF", k, "max |a-b| = %.3e" % d)
    print("bit-identical" if not bad else "%d of %d arrays differ" % (len(bad), len(a.files)))
    sys.exit(1 if bad else 0)

import synth  # noqa: E402
import paper_2106_12485_b200 as z  # noqa: E402

name, steps, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
cfg = synth.config(name)
sim = z.Simulation(cfg, inject=True)
hist = []
for n in range(steps):
    sim.step(1)
    it, fe, ke = sim.energy()
    hist.append([fe] + list(ke))
np.savez(out, E=sim.fields(0), B=sim.fields(1), J=sim.fields(2), energy=np.array(hist),
         particles=np.array([sim.counters()["particles"]]))
print(name, steps, "particles", sim.counters()["particles"])
