cd $GRAFT_REPO_ROOT
timeout 300 compute-sanitizer --print-limit 5 python -c "
import sys; sys.path.insert(0,'.')
import synth, paper_2106_12485_b200 as z
cfg = synth.config('C1', nx=48, ny=40)
sim = z.Simulation(cfg, inject=True)
sim.step(1); sim.sync(); print('ok')
" 2>&1 | head -40
