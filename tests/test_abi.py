"""The C-ABI library loads and exports every function include/zpic.h declares (no GPU
needed, no compute calls).  Also: the product package never imports the oracle."""
import ctypes
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build_module():
    """paper_2106_12485_b200/build.py loaded by path (the package itself refuses to import until
    the library exists), so the CPU suite also runs on a fresh checkout."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("_zpic_build", os.path.join(ROOT, "paper_2106_12485_b200", "build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def declared():
    src = open(os.path.join(ROOT, "include", "zpic.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:zpic_status|void|const char\*)\s+(zpic_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_five_calls():
    names = declared()
    for n in ("zpic_init", "zpic_step", "zpic_get_fields", "zpic_get_particles", "zpic_energy", "zpic_free"):
        assert n in names


def test_library_exports_every_declared_symbol():
    so = _build_module().build()
    lib = ctypes.CDLL(so)
    for n in declared():
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(zpic_\w+)", out))
    assert set(declared()) <= exported
    import paper_2106_12485_b200 as z
    assert set(z.EXPORTED) == set(declared())


def test_library_is_sm100a():
    so = _build_module().build()
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


def test_ctypes_structs_match_the_header(tmp_path):
    """The binding's ctypes mirrors of the ABI structs have the C compiler's size and field
    offsets (a silent mismatch would corrupt every argument block)."""
    _build_module().build()
    import paper_2106_12485_b200 as z
    structs = {name: getattr(z.zpic, name) for name in ("zpic_grid", "zpic_boundaries", "zpic_species",
                                                          "zpic_options", "zpic_dist")}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "zpic.h"', "int main(void) {"]
    for name, cls in structs.items():
        lines.append('printf("%s size %%zu\\n", sizeof(%s));' % (name, name))
        for f in cls._fields_:
            lines.append('printf("%s.%s %%zu\\n", offsetof(%s, %s));' % (name, f[0], name, f[0]))
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)])
    got = dict(l.rsplit(" ", 1) for l in subprocess.run([str(exe)], capture_output=True, text=True).stdout.splitlines())
    for name, cls in structs.items():
        assert int(got["%s size" % name]) == ctypes.sizeof(cls), name
        for f in cls._fields_:
            assert int(got["%s.%s" % (name, f[0])]) == getattr(cls, f[0]).offset, (name, f[0])


def test_enum_constants_match_the_header(tmp_path):
    """The binding's enum constants (boundaries, density profiles, transports) are the header's."""
    _build_module().build()
    import paper_2106_12485_b200 as z
    zz = z.zpic
    consts = {"ZPIC_BC_PERIODIC": zz.BC_PERIODIC, "ZPIC_BC_OPEN": zz.BC_OPEN,
              "ZPIC_BC_MOVING_WINDOW": zz.BC_MOVING_WINDOW, "ZPIC_TRANSPORT_NCCL": zz.TRANSPORT_NCCL,
              "ZPIC_TRANSPORT_LOOPBACK": zz.TRANSPORT_LOOPBACK, "ZPIC_TRANSPORT_PEER": zz.TRANSPORT_PEER,
              "ZPIC_TRANSPORT_LOOPBACK_PEER": zz.TRANSPORT_LOOPBACK_PEER}
    lines = ['#include <stdio.h>', '#include "zpic.h"', "int main(void) {"]
    lines += ['printf("%s %%d\\n", (int)%s);' % (k, k) for k in consts]
    lines.append("return 0; }")
    src = tmp_path / "enums.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "enums"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)])
    got = dict(l.rsplit(" ", 1) for l in subprocess.run([str(exe)], capture_output=True, text=True).stdout.splitlines())
    for k, v in consts.items():
        assert int(got[k]) == v, k
    assert set(zz.TRANSPORTS.values()) == {zz.TRANSPORT_NCCL, zz.TRANSPORT_LOOPBACK, zz.TRANSPORT_PEER,
                                          zz.TRANSPORT_LOOPBACK_PEER}


def _init_status(cfg, profile_override=None):
    """zpic_init's status for a config; the argument checks run before any device call, so this
    needs no GPU (a config that passes them would go on to touch the device: not used here)."""
    _build_module().build()
    import paper_2106_12485_b200 as z
    zz = z.zpic
    sps = []
    for s in cfg["species"]:
        prof = {"uniform": zz.DENS_UNIFORM, "slab": zz.DENS_SLAB, "ramp": zz.DENS_RAMP}[s.get("profile", "uniform")]
        sps.append(zz.zpic_species(s["m_q"], (ctypes.c_int32 * 2)(*s["ppc"]), s["n"], prof, s.get("x0", 0.0),
                                   s.get("x1", 0.0), (ctypes.c_double * 3)(*s["ufl"]), (ctypes.c_double * 3)(*s["uth"])))
    ctx = ctypes.c_void_p()
    arr = (zz.zpic_species * len(sps))(*sps)
    return zz._lib.zpic_init(ctypes.byref(ctx), ctypes.byref(zz.zpic_grid(cfg["nx"], cfg["ny"], cfg["dx"], cfg["dy"])),
                             cfg["dt"], arr, len(sps), ctypes.byref(zz.zpic_boundaries(*cfg["bc"])), 1, None, None)


def test_init_rejects_invalid_configs_before_touching_the_device():
    """zpic_init's documented errors (include/zpic.h): CFL, bad grid, bad species, and the
    moving-window injection reading R15 (a slab profile, or a ramp reaching past the box, has no
    defined density for the entering columns)."""
    import synth
    c4 = synth.config("C4")
    slab = synth.config("C4")
    slab["species"][0].update(profile="slab", x0=1.0, x1=50.0)
    far = synth.config("C4")
    far["species"][0].update(x0=70.0, x1=90.0)            # ends beyond Lx = 80
    cfl = synth.config("C1", dt=0.0708)                    # 1/sqrt(2)/10 = 0.07071
    tiny = synth.config("C1", nx=1)
    bad_ppc = synth.config("C1")
    bad_ppc["species"][0]["ppc"] = (0, 4)
    import paper_2106_12485_b200 as z
    assert _init_status(slab) == -1 and "R15" in z.zpic_last_error()
    assert _init_status(far) == -1 and "R15" in z.zpic_last_error()
    assert _init_status(cfl) == -2
    assert _init_status(tiny) == -1
    assert _init_status(bad_ppc) == -1
    assert c4["species"][0]["x1"] <= c4["nx"] * c4["dx"]   # the configs themselves satisfy R15
