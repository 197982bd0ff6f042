"""Thin ctypes binding of include/zpic.h (argument marshalling only; every stage of the step
runs in the CUDA kernels of libzpic_b200.so).  Function names match the C ABI.

There is no CPU fallback: importing this module without the built library raises.
PyTorch supplies device memory (its caching allocator, through the allocator hooks) and the
CUDA stream the library enqueues on.
"""
import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# ZPIC_SO: another in-tree build of the same library (same-box A/B timing of kernel variants,
# tools/gpu/ab.sh); only a bare file name inside this package directory is accepted
SO = os.path.join(HERE, os.path.basename(os.environ.get("ZPIC_SO", "libzpic_b200.so")))

if not os.path.exists(SO):
    raise ImportError("libzpic_b200.so is not built (run `python -m paper_2106_12485_b200.build` or "
                      "__graft_entry__.build()); there is no CPU fallback")
_lib = ctypes.CDLL(SO)

# ---- enums / structs (mirror include/zpic.h) ---------------------------------------------
ZPIC_OK = 0
STATUS = {0: "ZPIC_OK", -1: "ZPIC_E_INVALID", -2: "ZPIC_E_CFL", -3: "ZPIC_E_EMPTY_GRID", -4: "ZPIC_E_DECOMP",
          -5: "ZPIC_E_LASER", -6: "ZPIC_E_OOM", -7: "ZPIC_E_CUDA", -8: "ZPIC_E_NCCL", -9: "ZPIC_E_OVERFLOW",
          -10: "ZPIC_E_MIGRATION", -11: "ZPIC_E_BUFSIZE", -12: "ZPIC_E_STATE"}
BC_PERIODIC, BC_OPEN, BC_MOVING_WINDOW = 0, 1, 2
DENS_UNIFORM, DENS_SLAB, DENS_NONE, DENS_RAMP = 0, 1, 2, 3


class zpic_grid(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("dx", ctypes.c_double), ("dy", ctypes.c_double)]


class zpic_boundaries(ctypes.Structure):
    _fields_ = [("x", ctypes.c_int), ("y", ctypes.c_int)]


class zpic_species(ctypes.Structure):
    _fields_ = [("m_q", ctypes.c_double), ("ppc", ctypes.c_int32 * 2), ("n", ctypes.c_double), ("profile", ctypes.c_int),
                ("x0", ctypes.c_double), ("x1", ctypes.c_double), ("ufl", ctypes.c_double * 3),
                ("uth", ctypes.c_double * 3)]


ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p)


class zpic_options(ctypes.Structure):
    _fields_ = [("filter_passes", ctypes.c_int32), ("filter_compensated", ctypes.c_int32),
                ("track_ids", ctypes.c_int32), ("tile", ctypes.c_int32 * 2), ("capacity_slack", ctypes.c_double),
                ("mover_fraction", ctypes.c_double), ("profile", ctypes.c_int32), ("stream", ctypes.c_void_p),
                ("alloc", ALLOC_FN), ("free", FREE_FN), ("alloc_user", ctypes.c_void_p),
                ("current_mode", ctypes.c_int32), ("laser", ctypes.c_int32), ("laser_a0", ctypes.c_double),
                ("laser_omega0", ctypes.c_double), ("laser_fwhm", ctypes.c_double), ("laser_W0", ctypes.c_double),
                ("laser_start", ctypes.c_double), ("no_graphs", ctypes.c_int32),
                ("current_precision", ctypes.c_int32), ("halo_particles", ctypes.c_int32)]


TRANSPORT_NCCL, TRANSPORT_LOOPBACK, TRANSPORT_PEER, TRANSPORT_LOOPBACK_PEER = 0, 1, 2, 3
TRANSPORTS = {"nccl": TRANSPORT_NCCL, "loopback": TRANSPORT_LOOPBACK, "peer": TRANSPORT_PEER,
              "loopback_peer": TRANSPORT_LOOPBACK_PEER}


class zpic_dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("nccl_comm", ctypes.c_void_p),
                ("device", ctypes.c_int32), ("nccl_id", ctypes.c_void_p), ("transport", ctypes.c_int)]


_P = ctypes.c_void_p
_I32P = ctypes.POINTER(ctypes.c_int32)
_U32P = ctypes.POINTER(ctypes.c_uint32)
_F32P = ctypes.POINTER(ctypes.c_float)
_I64P = ctypes.POINTER(ctypes.c_int64)
_F64P = ctypes.POINTER(ctypes.c_double)

_lib.zpic_init.argtypes = [ctypes.POINTER(_P), ctypes.POINTER(zpic_grid), ctypes.c_double, ctypes.POINTER(zpic_species),
                           ctypes.c_int32, ctypes.POINTER(zpic_boundaries), ctypes.c_uint64, ctypes.POINTER(zpic_options),
                           ctypes.POINTER(zpic_dist)]
_lib.zpic_set_particles.argtypes = [_P, ctypes.c_int32, ctypes.c_int64, _I32P, _I32P, _F32P, _F32P, _F32P, _F32P, _F32P,
                                    _U32P]
_lib.zpic_set_fields.argtypes = [_P, ctypes.c_int32, _F32P, ctypes.c_size_t]
_lib.zpic_step.argtypes = [_P, ctypes.c_int32]
_lib.zpic_sync.argtypes = [_P]
_lib.zpic_get_fields.argtypes = [_P, ctypes.c_int32, _F32P, ctypes.c_size_t]
_lib.zpic_get_charge.argtypes = [_P, _F32P, ctypes.c_size_t]
_lib.zpic_get_particles.argtypes = [_P, ctypes.c_int32, _I64P, _I32P, _I32P, _F32P, _F32P, _F32P, _F32P, _F32P, _U32P]
_lib.zpic_energy.argtypes = [_P, _I64P, _F64P, _F64P]
_lib.zpic_layout.argtypes = [_P, _I32P, _I32P]
_lib.zpic_counters.argtypes = [_P, _I64P, ctypes.c_int32]
_lib.zpic_kernel_times.argtypes = [_P, ctypes.POINTER(ctypes.c_char_p), _F64P, _I32P, _I32P]
_lib.zpic_step_group.argtypes = [ctypes.POINTER(_P), ctypes.c_int32, ctypes.c_int32]
_lib.zpic_nccl_unique_id.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
_lib.zpic_peer_selftest.argtypes = [ctypes.c_int32] * 7 + [ctypes.c_int64, ctypes.c_int32, _I64P]
_lib.zpic_free.argtypes = [_P]
_lib.zpic_free.restype = None
_lib.zpic_last_error.argtypes = [_P]
_lib.zpic_last_error.restype = ctypes.c_char_p
for _f in ("zpic_init", "zpic_set_particles", "zpic_set_fields", "zpic_step", "zpic_sync", "zpic_get_fields",
           "zpic_get_particles", "zpic_energy", "zpic_layout", "zpic_counters", "zpic_kernel_times",
           "zpic_step_group", "zpic_nccl_unique_id", "zpic_peer_selftest"):
    getattr(_lib, _f).restype = ctypes.c_int

EXPORTED = ["zpic_init", "zpic_set_particles", "zpic_set_fields", "zpic_step", "zpic_step_group", "zpic_sync",
            "zpic_get_fields", "zpic_get_charge", "zpic_get_particles", "zpic_energy", "zpic_layout", "zpic_counters",
            "zpic_kernel_times", "zpic_nccl_unique_id", "zpic_peer_selftest", "zpic_free", "zpic_last_error"]


class ZpicError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("%s: %s" % (STATUS.get(status, status), msg))
        self.status = status


def _check(st, ctx=None):
    if st != ZPIC_OK:
        msg = _lib.zpic_last_error(ctx)
        raise ZpicError(st, msg.decode() if msg else "")


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptr(a, t):
    return a.ctypes.data_as(t) if a is not None else None


# ---- the ABI calls, one to one -------------------------------------------------------------
def zpic_init(grid, dt, species, bc, seed, options=None, dist=None):
    ctx = _P()
    sp = (zpic_species * max(1, len(species)))(*species)
    st = _lib.zpic_init(ctypes.byref(ctx), ctypes.byref(grid), dt, sp, len(species), ctypes.byref(bc), seed,
                        ctypes.byref(options) if options is not None else None,
                        ctypes.byref(dist) if dist is not None else None)
    _check(st, None)
    return ctx


def zpic_set_particles(ctx, species, ix, iy, x, y, ux, uy, uz, id=None):
    ix = np.ascontiguousarray(ix, dtype=np.int32)
    iy = np.ascontiguousarray(iy, dtype=np.int32)
    x, y, ux, uy, uz = (_f32(a) for a in (x, y, ux, uy, uz))
    idv = np.ascontiguousarray(id, dtype=np.uint32) if id is not None else None
    _check(_lib.zpic_set_particles(ctx, species, len(ix), _ptr(ix, _I32P), _ptr(iy, _I32P), _ptr(x, _F32P),
                                   _ptr(y, _F32P), _ptr(ux, _F32P), _ptr(uy, _F32P), _ptr(uz, _F32P),
                                   _ptr(idv, _U32P)), ctx)


def zpic_set_fields(ctx, which, arr):
    a = _f32(arr)
    _check(_lib.zpic_set_fields(ctx, which, _ptr(a, _F32P), a.size), ctx)


def zpic_step(ctx, n):
    _check(_lib.zpic_step(ctx, n), ctx)


def zpic_step_group(ctxs, n):
    arr = (_P * len(ctxs))(*[c.value if isinstance(c, _P) else c for c in ctxs])
    st = _lib.zpic_step_group(arr, len(ctxs), n)
    _check(st, ctxs[0])


def zpic_nccl_unique_id():
    buf = ctypes.create_string_buffer(128)
    _check(_lib.zpic_nccl_unique_id(buf, 128), None)
    return buf.raw


def zpic_peer_selftest(ranks, epochs, nx, ny, pcap, periodic=True, commutative=False, budget_cycles=4_000_000_000,
                       fault=0):
    """The PEER protocol self-test (include/zpic.h): returns (mismatched values, timed-out waits)."""
    err = ctypes.c_int64(0)
    _check(_lib.zpic_peer_selftest(ranks, epochs, nx, ny, pcap, 1 if periodic else 0, 1 if commutative else 0,
                                   budget_cycles, fault, ctypes.byref(err)), None)
    return err.value & ((1 << 40) - 1), err.value >> 40


def zpic_sync(ctx):
    _check(_lib.zpic_sync(ctx), ctx)


def zpic_layout(ctx):
    y0, ny = ctypes.c_int32(), ctypes.c_int32()
    _check(_lib.zpic_layout(ctx, ctypes.byref(y0), ctypes.byref(ny)), ctx)
    return y0.value, ny.value


def zpic_get_fields(ctx, which, nx, ny_local, out=None):
    if out is None:
        out = np.empty((3, ny_local, nx), dtype=np.float32)
    _check(_lib.zpic_get_fields(ctx, which, _ptr(out, _F32P), out.size), ctx)
    return out


def zpic_get_charge(ctx, nx, ny_local, out=None):
    if out is None:
        out = np.empty((ny_local, nx), dtype=np.float32)
    _check(_lib.zpic_get_charge(ctx, _ptr(out, _F32P), out.size), ctx)
    return out


def zpic_get_particles(ctx, species, with_id=False):
    n = ctypes.c_int64(0)
    _check(_lib.zpic_get_particles(ctx, species, ctypes.byref(n), None, None, None, None, None, None, None, None), ctx)
    N = n.value
    ix = np.empty(N, np.int32); iy = np.empty(N, np.int32)
    f = [np.empty(N, np.float32) for _ in range(5)]
    idv = np.empty(N, np.uint32) if with_id else None
    _check(_lib.zpic_get_particles(ctx, species, ctypes.byref(n), _ptr(ix, _I32P), _ptr(iy, _I32P),
                                   *[_ptr(a, _F32P) for a in f], _ptr(idv, _U32P)), ctx)
    d = {"ix": ix, "iy": iy, "x": f[0], "y": f[1], "ux": f[2], "uy": f[3], "uz": f[4]}
    if with_id:
        d["id"] = idv
    return d


def zpic_energy(ctx, nspecies):
    it = ctypes.c_int64()
    fe = ctypes.c_double()
    ke = (ctypes.c_double * 4)()
    _check(_lib.zpic_energy(ctx, ctypes.byref(it), ctypes.byref(fe), ke), ctx)
    return it.value, fe.value, [ke[s] for s in range(nspecies)]


def zpic_counters(ctx):
    out = (ctypes.c_int64 * 11)()
    _check(_lib.zpic_counters(ctx, out, 11), ctx)
    keys = ("particles", "movers", "max_fill_permille", "repacks", "steps", "tiles", "launches", "tile",
            "sorted_tiles", "unsorted_tiles", "loose")
    return dict(zip(keys, list(out)))


def zpic_kernel_times(ctx):
    n = ctypes.c_int32(16)
    names = (ctypes.c_char_p * 16)()
    ms = (ctypes.c_double * 16)()
    cnt = (ctypes.c_int32 * 16)()
    _check(_lib.zpic_kernel_times(ctx, names, ms, cnt, ctypes.byref(n)), ctx)
    return {names[k].decode(): (ms[k], cnt[k]) for k in range(n.value)}


def zpic_free(ctx):
    _lib.zpic_free(ctx)


def zpic_last_error(ctx=None):
    m = _lib.zpic_last_error(ctx)
    return m.decode() if m else ""


# ---- convenience wrapper ------------------------------------------------------------------
class Simulation:
    """A context built from a config dict (the layout of synth/configs.py: nx, ny, dx, dy, dt,
    bc, seed, species[m_q, ppc, n, profile, x0, x1, ufl, uth], filter).  With inject=True the
    species are injected on the device (uniform / slab profiles); otherwise call
    set_particles.  Device memory comes from PyTorch's caching allocator and work goes on
    PyTorch's current CUDA stream when torch_plumbing is True."""

    def __init__(self, cfg, inject=True, track_ids=False, tile=16, profile=False, capacity_slack=1.25,
                 torch_plumbing=True, stream=None, dist=None, current_mode=0, graphs=True, current_precision=0):
        """dist: None (whole domain) or {"rank", "world", "transport": "nccl" | "loopback" | "peer" | "loopback_peer",
        "nccl_id": 128 bytes | "nccl_comm": ncclComm_t address} (y-slab decomposition)."""
        self.cfg = cfg
        self.nx, self.ny = cfg["nx"], cfg["ny"]
        self.nspecies = len(cfg["species"])
        grid = zpic_grid(cfg["nx"], cfg["ny"], cfg["dx"], cfg["dy"])
        bc = zpic_boundaries(*cfg["bc"])
        sps = []
        for s in cfg["species"]:
            prof = {"uniform": DENS_UNIFORM, "slab": DENS_SLAB, "ramp": DENS_RAMP}.get(s.get("profile", "uniform"),
                                                                                    DENS_NONE)
            if not inject:
                prof = DENS_NONE
            sps.append(zpic_species(s["m_q"], (ctypes.c_int32 * 2)(*s["ppc"]), s["n"], prof, s.get("x0", 0.0),
                                    s.get("x1", 0.0), (ctypes.c_double * 3)(*s["ufl"]),
                                    (ctypes.c_double * 3)(*s["uth"])))
        filt = cfg.get("filter", (0, 0))
        opt = zpic_options()
        opt.filter_passes, opt.filter_compensated = filt
        opt.track_ids = int(track_ids)
        opt.tile[0] = opt.tile[1] = tile
        opt.capacity_slack = capacity_slack
        opt.mover_fraction = 0.05
        opt.profile = int(profile)
        opt.current_mode = int(current_mode)
        opt.no_graphs = 0 if graphs else 1
        opt.current_precision = {"auto": 0, "exact": 1}.get(current_precision, current_precision)
        if inject and "laser" in cfg:     # the laser initial fields (R17) on the device
            las = cfg["laser"]
            if las.get("polarization", "y") != "y":
                raise ValueError("only a y-polarised laser is implemented (R17)")
            opt.laser = 1
            opt.laser_a0, opt.laser_omega0, opt.laser_fwhm = las["a0"], las["omega0"], las["fwhm"]
            opt.laser_W0, opt.laser_start = las["W0"], las["start"]
        self._keep = []
        if torch_plumbing:
            import torch
            dev = torch.cuda.current_device()
            st = stream if stream is not None else torch.cuda.current_stream()
            if st.cuda_stream == 0:      # the legacy NULL stream: give the library a real one
                st = torch.cuda.Stream()
            opt.stream = st.cuda_stream
            self.torch_stream = st

            def _alloc(nbytes, user):
                return torch.cuda.caching_allocator_alloc(int(nbytes), dev, st)

            cad = torch.cuda.caching_allocator_delete

            def _free(ptr, user):
                try:
                    cad(ptr)
                except Exception:      # interpreter teardown: torch already gone, memory goes with the process
                    pass
            a, f = ALLOC_FN(_alloc), FREE_FN(_free)
            self._keep += [a, f]
            opt.alloc, opt.free = a, f
        dst = None
        if dist is not None:
            dst = zpic_dist()
            dst.rank, dst.world = dist["rank"], dist["world"]
            dst.transport = TRANSPORTS[dist.get("transport", "nccl")]
            dst.nccl_comm = dist.get("nccl_comm")
            self._nccl_id = ctypes.create_string_buffer(dist["nccl_id"], 128) if dist.get("nccl_id") else None
            dst.nccl_id = ctypes.cast(self._nccl_id, ctypes.c_void_p) if self._nccl_id is not None else None
            dst.device = dist.get("device", 0)
        self.dist = dist
        self.ctx = zpic_init(grid, cfg["dt"], sps, bc, cfg["seed"], opt, dst)
        self.y0, self.ny_local = zpic_layout(self.ctx)

    def set_particles(self, s, p):
        zpic_set_particles(self.ctx, s, p["ix"], p["iy"], p["x"], p["y"], p["ux"], p["uy"], p["uz"], p.get("id"))

    def set_fields(self, which, arr):
        zpic_set_fields(self.ctx, which, arr)

    def step(self, n=1):
        zpic_step(self.ctx, n)

    def sync(self):
        zpic_sync(self.ctx)

    def fields(self, which):
        y0, nyl = zpic_layout(self.ctx)
        return zpic_get_fields(self.ctx, which, self.nx, nyl)

    def charge(self):
        y0, nyl = zpic_layout(self.ctx)
        return zpic_get_charge(self.ctx, self.nx, nyl)

    def particles(self, s, with_id=False):
        return zpic_get_particles(self.ctx, s, with_id)

    def energy(self):
        return zpic_energy(self.ctx, self.nspecies)

    def counters(self):
        return zpic_counters(self.ctx)

    def kernel_times(self):
        return zpic_kernel_times(self.ctx)

    def close(self):
        if self.ctx:
            zpic_free(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
