import sys; sys.path.insert(0, '.')
import synth, paper_2106_12485_b200 as z
cfg = synth.config("C5")
sim = z.Simulation(cfg, inject=True, tile=16)
import ctypes
out = (ctypes.c_int64 * 7)()
st = z.zpic._lib.zpic_counters(sim.ctx, out, 7)
print("status", st, z.zpic_last_error(sim.ctx), list(out))
