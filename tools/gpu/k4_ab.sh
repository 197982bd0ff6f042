# build the variants first: for r in 2 4 8 16; do python tools/build_variant.py k4r$r -DZPIC_K4R=$r; done
# Same-box A/B of K4 (k_assemble_j) rows per thread (libzpic_b200.k4rN.so, -DZPIC_K4R=N) at C5
for r in 1 2; do for v in ${VARIANTS:-k4r2 k4r4 k4r8 k4r16}; do
  ZPIC_SO=libzpic_b200.$v.so timeout 300 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 2>/dev/null | grep "^{" | python -c "
import sys, json
d = json.loads(sys.stdin.read()); k = d['kernel_ms_per_step']
print('%-6s ms/step %.4f K4 %.4f yee %.4f' % ('$v', d['ms_per_step'], k['k_assemble_j'], k['k_yee']))"
done; done
