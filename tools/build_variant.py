"""Build an in-tree variant of libzpic_b200.so with extra nvcc flags (same-box A/B timing:
ZPIC_SO=libzpic_b200.<tag>.so selects it, tools/gpu/ab.sh / ab2.sh interleave the variants).
usage: python tools/build_variant.py TAG [-DFLAG ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2106_12485_b200"))
import build  # noqa: E402

tag, flags = sys.argv[1], sys.argv[2:]
build.SO = os.path.join(build.HERE, "libzpic_b200.%s.so" % tag)
build.FLAGS = build.FLAGS + flags
print(build.build(force=True))
