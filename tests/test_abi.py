"""The C-ABI library loads and exports every function include/zpic.h declares (no GPU
needed, no compute calls).  Also: the product package never imports the oracle."""
import ctypes
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "zpic.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:zpic_status|void|const char\*)\s+(zpic_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_five_calls():
    names = declared()
    for n in ("zpic_init", "zpic_step", "zpic_get_fields", "zpic_get_particles", "zpic_energy", "zpic_free"):
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_2106_12485_b200 import build
    so = build.build()
    lib = ctypes.CDLL(so)
    for n in declared():
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(zpic_\w+)", out))
    assert set(declared()) <= exported
    import paper_2106_12485_b200 as z
    assert set(z.EXPORTED) == set(declared())


def test_library_is_sm100a():
    from paper_2106_12485_b200 import build
    so = build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2106_12485_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", txt, flags=re.M), f
                assert "zpic_oracle" not in txt and "liborc" not in txt, f
