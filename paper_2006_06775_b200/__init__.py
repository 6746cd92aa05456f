"""Thin Python binding of libbdm.so (include/bdm.h) -- argument marshalling only.

Every step of the mechanical-interaction path runs in the CUDA kernels of libbdm.so; this module
never computes any part of it and has no fallback: if the library is missing or no CUDA device
is present, the calls raise.

Functions carry the C names (bdm_init, bdm_grid_build, bdm_mech_step, bdm_get_displacements, ...).
Arrays may be NumPy arrays (host; copied by the library) or CUDA torch tensors (passed as device
pointers with BDM_DEVICE_PTRS on the handle's stream).
"""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB_PATH = os.environ.get("BDM_LIBRARY") or os.path.join(HERE, "libbdm.so")  # override: kernel-variant experiments
HEADER = os.path.join(ROOT, "include", "bdm.h")

BDM_OK = 0
BDM_EINVAL = -1
BDM_ESTATE = -2
BDM_ENOMEM = -3
BDM_ECUDA = -4
BDM_ENCCL = -5
BDM_ENONFINITE = -6
BDM_ERANGE = -7
BDM_ETRUNC = -8
BDM_DEVICE_PTRS = 0x1
BDM_RECORD = 0x2
BDM_SKIP_STATIONARY = 0x4
BDM_NEIGHBOR = 0
BDM_CONTACT = 1
BDM_HALO = 0
BDM_MIGRANTS = 1
BDM_OWNED_POSITIONS = 0
BDM_LAST_DISPLACEMENTS = 1
BDM_PATH_AUTO = 0
BDM_PATH_SINGLE = 1

ERRNAMES = {-1: "EINVAL", -2: "ESTATE", -3: "ENOMEM", -4: "ECUDA", -5: "ENCCL", -6: "ENONFINITE", -7: "ERANGE",
            -8: "ETRUNC"}


class BdmError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"BDM_{ERRNAMES.get(code, code)}: {msg}")
        self.code = code


class bdm_params(ctypes.Structure):
    _fields_ = [("k_rep", ctypes.c_double), ("gamma_att", ctypes.c_double), ("adherence", ctypes.c_double),
                ("dt", ctypes.c_double), ("eta", ctypes.c_double), ("max_disp", ctypes.c_double),
                ("box_edge_min", ctypes.c_double), ("flags", ctypes.c_uint32), ("device", ctypes.c_int32)]


class bdm_grid_info(ctypes.Structure):
    _fields_ = [("L", ctypes.c_double), ("L2", ctypes.c_double), ("inv", ctypes.c_double),
                ("lo", ctypes.c_int32 * 3), ("hi", ctypes.c_int32 * 3), ("n_boxes", ctypes.c_int64),
                ("n_agents", ctypes.c_int64)]


class bdm_field_params(ctypes.Structure):
    _fields_ = [("h", ctypes.c_double), ("origin", ctypes.c_double * 3), ("dims", ctypes.c_int32 * 3),
                ("diff", ctypes.c_double), ("decay", ctypes.c_double), ("dt", ctypes.c_double),
                ("secretion", ctypes.c_double), ("speed", ctypes.c_double)]


class bdm_stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("n_agents", "steps", "launches", "host_syncs", "half_path", "migrated",
                                               "ghosts", "exchange_bytes", "chunks", "redo_chunks", "world",
                                               "local_ranks")]


class bdm_agent_stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("n_cand", "n_nb", "n_ct", "branch", "nb_hash", "ct_hash")]


_vp = ctypes.c_void_p
_SIGS = {
    "bdm_abi_version": ([], ctypes.c_int),
    "bdm_params_default": ([ctypes.POINTER(bdm_params)], ctypes.c_int),
    "bdm_init": ([ctypes.POINTER(_vp), ctypes.c_int64, _vp, _vp, ctypes.POINTER(bdm_params)], ctypes.c_int),
    "bdm_grid_build": ([_vp], ctypes.c_int),
    "bdm_mech_step": ([_vp, ctypes.c_int32], ctypes.c_int),
    "bdm_get_displacements": ([_vp, _vp], ctypes.c_int),
    "bdm_get_positions": ([_vp, _vp], ctypes.c_int),
    "bdm_get_box_coords": ([_vp, _vp], ctypes.c_int),
    "bdm_get_diameters": ([_vp, _vp], ctypes.c_int),
    "bdm_get_grid_info": ([_vp, ctypes.POINTER(bdm_grid_info)], ctypes.c_int),
    "bdm_get_agent_stats": ([_vp, ctypes.POINTER(bdm_agent_stats)], ctypes.c_int),
    "bdm_get_pairs": ([_vp, ctypes.c_int, ctypes.POINTER(ctypes.c_int64), _vp, ctypes.c_int64], ctypes.c_int),
    "bdm_set_agents": ([_vp, _vp, _vp], ctypes.c_int),
    "bdm_get_skip_stats": ([_vp, _vp], ctypes.c_int),
    "bdm_get_path_stats": ([_vp, _vp], ctypes.c_int),
    "bdm_set_growth": ([_vp, ctypes.c_double, ctypes.c_double, ctypes.c_uint64], ctypes.c_int),
    "bdm_reserve": ([_vp, ctypes.c_int64], ctypes.c_int),
    "bdm_set_neurites": ([_vp, ctypes.c_int64, _vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_double], ctypes.c_int),
    "bdm_get_neurites": ([_vp, _vp, _vp], ctypes.c_int),
    "bdm_set_fields": ([_vp, ctypes.POINTER(bdm_field_params), _vp], ctypes.c_int),
    "bdm_get_field": ([_vp, ctypes.c_int, _vp], ctypes.c_int),
    "bdm_get_count": ([_vp, _vp], ctypes.c_int),
    "bdm_set_stream": ([_vp, _vp], ctypes.c_int),
    "bdm_sync": ([_vp], ctypes.c_int),
    "bdm_set_timing": ([_vp, ctypes.c_int], ctypes.c_int),
    "bdm_set_defer": ([_vp, ctypes.c_int], ctypes.c_int),
    "bdm_set_force_path": ([_vp, ctypes.c_int], ctypes.c_int),
    "bdm_get_timing": ([_vp, _vp], ctypes.c_int),
    "bdm_get_timing_ex": ([_vp, _vp], ctypes.c_int),
    "bdm_generate_uniform": ([ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, _vp, _vp, ctypes.c_double,
                              ctypes.c_double, _vp, _vp, _vp], ctypes.c_int),
    "bdm_slab_init": ([ctypes.POINTER(_vp), ctypes.c_int64, ctypes.c_int64, _vp, _vp, _vp,
                       ctypes.POINTER(bdm_params)], ctypes.c_int),
    "bdm_slab_load": ([_vp, ctypes.c_int64, _vp, _vp, _vp], ctypes.c_int),
    "bdm_slab_local_maxd": ([_vp, ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
    "bdm_slab_set_box_edge": ([_vp, ctypes.c_double], ctypes.c_int),
    "bdm_slab_local_extents": ([_vp, _vp], ctypes.c_int),
    "bdm_slab_pack": ([_vp, ctypes.c_int, ctypes.c_int32, ctypes.c_int32, _vp, _vp, ctypes.c_int64,
                       ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)], ctypes.c_int),
    "bdm_slab_add": ([_vp, _vp, ctypes.c_int64, _vp, ctypes.c_int64], ctypes.c_int),
    "bdm_slab_split": ([_vp, ctypes.c_int32, ctypes.c_int32, _vp, _vp, ctypes.c_int64, _vp], ctypes.c_int),
    "bdm_slab_commit": ([_vp, ctypes.c_int64], ctypes.c_int),
    "bdm_slab_step": ([_vp, _vp, _vp, ctypes.c_int32, ctypes.c_int32, _vp, ctypes.c_int64, _vp, ctypes.c_int64,
                       ctypes.c_int], ctypes.c_int),
    "bdm_slab_get": ([_vp, ctypes.c_int, ctypes.POINTER(ctypes.c_int64), _vp, _vp], ctypes.c_int),
    "bdm_nccl_unique_id": ([_vp], ctypes.c_int),
    "bdm_init_dist": ([ctypes.POINTER(_vp), ctypes.c_int64, _vp, _vp, _vp, ctypes.POINTER(bdm_params), ctypes.c_int,
                       ctypes.c_int, _vp, ctypes.c_int, _vp], ctypes.c_int),
    "bdm_init_dist_local": ([ctypes.POINTER(_vp), ctypes.c_int, _vp, _vp, _vp, _vp, ctypes.POINTER(bdm_params), _vp],
                            ctypes.c_int),
    "bdm_get_local": ([_vp, ctypes.c_int, ctypes.POINTER(ctypes.c_int64), _vp, _vp], ctypes.c_int),
    "bdm_set_agents_dist": ([_vp, ctypes.c_int64, _vp, _vp, _vp], ctypes.c_int),
    "bdm_get_cuts": ([_vp, _vp, ctypes.c_int32], ctypes.c_int),
    "bdm_get_pair_digest": ([_vp, ctypes.c_int, _vp, _vp], ctypes.c_int),
    "bdm_get_stats": ([_vp, ctypes.POINTER(bdm_stats)], ctypes.c_int),
    "bdm_last_error": ([_vp], ctypes.c_char_p),
    "bdm_destroy": ([_vp], None),
}

_lib = None


def load_library():
    """Load libbdm.so (raises if it has not been built: there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `make` or __graft_entry__.build() first")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
    return _lib


def header_symbols(path: str = HEADER) -> list[str]:
    """Function names declared in include/bdm.h."""
    txt = open(path).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(bdm_\w+)\s*\(", txt, flags=re.M)))


def _check(rc: int, h=None):
    if rc != BDM_OK:
        msg = load_library().bdm_last_error(h)
        raise BdmError(rc, msg.decode() if msg else "")


def bdm_params_default(**overrides) -> bdm_params:
    p = bdm_params()
    _check(load_library().bdm_params_default(ctypes.byref(p)))
    for k, v in overrides.items():
        setattr(p, k, v)
    return p


def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


def _ptr(a):
    if a is None:
        return None
    if _is_torch(a):
        return ctypes.c_void_p(a.data_ptr())
    return ctypes.c_void_p(a.ctypes.data)


class _Sized:
    """View of a handle with another row count (for last-step outputs)."""

    def __init__(self, h, n):
        self.raw, self.n, self.device_ptrs = h.raw, n, h.device_ptrs


class Handle:
    """Owns a bdm_handle; destroyed with the object."""

    def __init__(self, raw: ctypes.c_void_p, n: int, device_ptrs: bool):
        self.raw = raw
        self.n = n
        self.device_ptrs = device_ptrs

    def __del__(self):
        if getattr(self, "raw", None) and _lib is not None:
            _lib.bdm_destroy(self.raw)
            self.raw = None

    def close(self):
        self.__del__()


def bdm_init(pos, diam, params: bdm_params | None = None, stream=None) -> Handle:
    """pos [n,3] fp64 and diam [n] fp64, NumPy (host) or CUDA torch tensors (device pointers)."""
    lib = load_library()
    p = params if params is not None else bdm_params_default()
    dev = _is_torch(pos) and pos.is_cuda
    if dev:
        import torch

        assert pos.dtype == torch.float64 and diam.dtype == torch.float64 and pos.is_contiguous()
        p.flags |= BDM_DEVICE_PTRS
        if p.device < 0:
            p.device = pos.device.index
        n = pos.shape[0]
    else:
        p.flags &= ~BDM_DEVICE_PTRS
        pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
        diam = np.ascontiguousarray(diam, dtype=np.float64).reshape(-1)
        n = pos.shape[0]
        if diam.shape[0] != n:
            raise ValueError("pos and diam lengths differ")
    raw = ctypes.c_void_p()
    if dev and stream is not None:
        # the copy kernel of bdm_init runs on the default stream; order it after the producer
        stream.synchronize()
    _check(lib.bdm_init(ctypes.byref(raw), n, _ptr(pos), _ptr(diam), ctypes.byref(p)))
    h = Handle(raw, n, dev)
    if stream is not None:
        bdm_set_stream(h, stream)
    return h


def bdm_set_agents(h: Handle, pos, diam) -> None:
    """Replace the population (same n); host arrays or CUDA tensors matching the handle's mode."""
    if not h.device_ptrs:
        pos = np.ascontiguousarray(pos, dtype=np.float64)
        diam = np.ascontiguousarray(diam, dtype=np.float64)
    _check(load_library().bdm_set_agents(h.raw, _ptr(pos), _ptr(diam)), h.raw)


def bdm_set_stream(h: Handle, stream) -> None:
    sp = getattr(stream, "cuda_stream", stream)
    _check(load_library().bdm_set_stream(h.raw, ctypes.c_void_p(sp)), h.raw)


def bdm_grid_build(h: Handle) -> None:
    _check(load_library().bdm_grid_build(h.raw), h.raw)


def bdm_mech_step(h: Handle, n_steps: int = 1) -> None:
    _check(load_library().bdm_mech_step(h.raw, n_steps), h.raw)
    bdm_get_count(h)


def bdm_sync(h: Handle) -> None:
    _check(load_library().bdm_sync(h.raw), h.raw)


def _out(h: Handle, shape, dtype, out):
    if out is not None:
        return out
    if h.device_ptrs:
        import torch

        tdt = {np.float64: torch.float64, np.int32: torch.int32, np.int8: torch.int8, np.uint64: torch.int64}[dtype]
        return torch.empty(shape, dtype=tdt, device="cuda")
    return np.empty(shape, dtype=dtype)


def bdm_get_count(h: Handle):
    """(current agents, agents of the last mechanics step)."""
    out = np.zeros(2, np.int64)
    _check(load_library().bdm_get_count(h.raw, _ptr(out)), h.raw)
    h.n = int(out[0])
    return int(out[0]), int(out[1])


def bdm_set_growth(h: Handle, growth: float, div_diam: float, seed: int = 0) -> None:
    _check(load_library().bdm_set_growth(h.raw, growth, div_diam, seed), h.raw)


def bdm_set_fields(h: Handle, h_spacing: float, origin, dims, diff: float, decay: float, dt: float,
                   secretion: float, speed: float, types) -> None:
    """Soma clustering (NEXT-3): two substance lattices + chemotaxis before each mechanics step."""
    fp = bdm_field_params(h_spacing, (ctypes.c_double * 3)(*origin), (ctypes.c_int32 * 3)(*dims), diff, decay, dt,
                          secretion, speed)
    if not h.device_ptrs:
        types = np.ascontiguousarray(types, dtype=np.int8)
    h.field_dims = tuple(int(d) for d in dims)
    _check(load_library().bdm_set_fields(h.raw, ctypes.byref(fp), _ptr(types)), h.raw)


def bdm_get_field(h: Handle, which: int, out=None):
    if out is None:
        if h.device_ptrs:
            import torch

            out = torch.empty(h.field_dims, dtype=torch.float64, device="cuda")
        else:
            out = np.empty(h.field_dims, np.float64)
    _check(load_library().bdm_get_field(h.raw, which, _ptr(out)), h.raw)
    return out


def bdm_set_neurites(h: Handle, distal, diam, rest_len, anchor, mother, daughters, k_spring: float) -> None:
    """NEXT-4: neurite elements (host arrays; element id = index; -1 = no mother / daughter)."""
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (distal, diam, rest_len, anchor)]
    m = np.ascontiguousarray(mother, dtype=np.int64)
    d = np.ascontiguousarray(daughters, dtype=np.int64).reshape(-1, 2)
    h.n_el = len(m)
    _check(load_library().bdm_set_neurites(h.raw, len(m), *(_ptr(a) for a in arrs), _ptr(m), _ptr(d), k_spring),
           h.raw)


def bdm_get_neurites(h: Handle):
    """(distal points [E,3], their displacements of the last step [E,3])."""
    E = getattr(h, "n_el", 0)
    q = np.zeros((E, 3))
    dq = np.zeros((E, 3))
    _check(load_library().bdm_get_neurites(h.raw, _ptr(q), _ptr(dq)), h.raw)
    return q, dq


def bdm_reserve(h: Handle, capacity: int) -> None:
    _check(load_library().bdm_reserve(h.raw, capacity), h.raw)


def bdm_get_displacements(h: Handle, out=None):
    _, n_dp = bdm_get_count(h)
    out = _out(h, (n_dp, 3), np.float64, out)
    _check(load_library().bdm_get_displacements(h.raw, _ptr(out)), h.raw)
    return out


def bdm_get_positions(h: Handle, out=None):
    bdm_get_count(h)
    out = _out(h, (h.n, 3), np.float64, out)
    _check(load_library().bdm_get_positions(h.raw, _ptr(out)), h.raw)
    return out


def bdm_get_diameters(h: Handle, out=None):
    bdm_get_count(h)
    out = _out(h, (h.n,), np.float64, out)
    _check(load_library().bdm_get_diameters(h.raw, _ptr(out)), h.raw)
    return out


def bdm_get_box_coords(h: Handle, out=None):
    out = _out(h, (h.n, 3), np.int32, out)
    _check(load_library().bdm_get_box_coords(h.raw, _ptr(out)), h.raw)
    return out


def bdm_get_grid_info(h: Handle) -> dict:
    g = bdm_grid_info()
    _check(load_library().bdm_get_grid_info(h.raw, ctypes.byref(g)), h.raw)
    return dict(L=g.L, L2=g.L2, inv=g.inv, lo=tuple(g.lo), hi=tuple(g.hi), n_boxes=g.n_boxes, n_agents=g.n_agents)


def bdm_get_agent_stats(h: Handle) -> dict:
    """Per-agent record of the last step (host NumPy arrays; requires BDM_RECORD)."""
    n_cur, n_dp = bdm_get_count(h)
    h = _Sized(h, n_dp or n_cur)
    if h.device_ptrs:
        import torch

        out = dict(n_cand=torch.empty(h.n, dtype=torch.int32, device="cuda"),
                   n_nb=torch.empty(h.n, dtype=torch.int32, device="cuda"),
                   n_ct=torch.empty(h.n, dtype=torch.int32, device="cuda"),
                   branch=torch.empty(h.n, dtype=torch.int8, device="cuda"),
                   nb_hash=torch.empty(h.n, dtype=torch.int64, device="cuda"),
                   ct_hash=torch.empty(h.n, dtype=torch.int64, device="cuda"))
    else:
        out = dict(n_cand=np.empty(h.n, np.int32), n_nb=np.empty(h.n, np.int32), n_ct=np.empty(h.n, np.int32),
                   branch=np.empty(h.n, np.int8), nb_hash=np.empty(h.n, np.uint64), ct_hash=np.empty(h.n, np.uint64))
    st = bdm_agent_stats(*(_ptr(out[k]).value for k in ("n_cand", "n_nb", "n_ct", "branch", "nb_hash", "ct_hash")))
    _check(load_library().bdm_get_agent_stats(h.raw, ctypes.byref(st)), h.raw)
    return out


def bdm_get_pairs(h: Handle, kind: int) -> np.ndarray:
    """Sorted unordered pairs (min id, max id) as int64 [P, 2] (host)."""
    lib = load_library()
    cnt = ctypes.c_int64(0)
    rc = lib.bdm_get_pairs(h.raw, kind, ctypes.byref(cnt), None, 0)
    if rc not in (BDM_OK, BDM_ETRUNC):
        _check(rc, h.raw)
    out = np.empty((max(cnt.value, 1), 2), np.int64)
    _check(lib.bdm_get_pairs(h.raw, kind, ctypes.byref(cnt), _ptr(out), cnt.value), h.raw)
    return out[: cnt.value]


def bdm_get_skip_stats(h: Handle) -> dict:
    """NEXT-1 statistics of the last step: agents moved, agents searched, N."""
    out = np.zeros(3, np.int64)
    _check(load_library().bdm_get_skip_stats(h.raw, _ptr(out)), h.raw)
    return dict(moved=int(out[0]), searched=int(out[1]), n=int(out[2]))


def bdm_get_path_stats(h: Handle) -> dict:
    """Force path of the last step: half-shell pair path used (1/0), agents that overflowed their
    pair rows and took the exact full-search path."""
    out = np.zeros(2, np.int64)
    _check(load_library().bdm_get_path_stats(h.raw, _ptr(out)), h.raw)
    return dict(half=int(out[0]), slow=int(out[1]))


def bdm_set_force_path(h: Handle, path: int) -> None:
    """BDM_PATH_AUTO (half-shell passes when their rows fit, else k_force) or BDM_PATH_SINGLE."""
    _check(load_library().bdm_set_force_path(h.raw, int(path)), h.raw)


def bdm_set_defer(h: Handle, max_deferred: int) -> None:
    """At most max_deferred consecutive deferred builds inside one bdm_mech_step call (0 = off)."""
    _check(load_library().bdm_set_defer(h.raw, int(max_deferred)), h.raw)


def bdm_set_timing(h: Handle, enabled: bool = True) -> None:
    _check(load_library().bdm_set_timing(h.raw, int(enabled)), h.raw)


def bdm_get_timing(h: Handle) -> dict:
    """Device ms of the grid-build and force kernels summed over the steps since the last call
    (force split into the half-shell search and sum passes where that path ran)."""
    out = np.zeros(6)
    _check(load_library().bdm_get_timing_ex(h.raw, _ptr(out)), h.raw)
    return dict(grid_ms=float(out[0]), force_ms=float(out[1]), steps=int(out[2]), launches=int(out[3]),
                search_ms=float(out[4]), sum_ms=float(out[5]))


def bdm_generate_uniform(seed: int, id0: int, n: int, lo3, hi3, dlo: float, dhi: float, pos, diam, stream=None):
    """Counter-hash population on the device (pos, diam are CUDA torch tensors)."""
    lo = np.ascontiguousarray(lo3, np.float64)
    hi = np.ascontiguousarray(hi3, np.float64)
    sp = getattr(stream, "cuda_stream", stream) if stream is not None else None
    _check(load_library().bdm_generate_uniform(seed, id0, n, _ptr(lo), _ptr(hi), dlo, dhi, _ptr(pos), _ptr(diam),
                                               ctypes.c_void_p(sp) if sp else None))


# ------------------------------------------------------------------------------------ x-slab mode
def bdm_slab_init(ids, pos, diam, capacity: int, params: bdm_params | None = None, stream=None) -> Handle:
    """ids uint32-compatible (torch.int32 / int64 converted), pos [n,3], diam [n]: CUDA tensors."""
    import torch

    lib = load_library()
    p = params if params is not None else bdm_params_default()
    p.flags |= BDM_DEVICE_PTRS
    if p.device < 0:
        p.device = pos.device.index
    n = pos.shape[0]
    ids32 = ids.to(torch.int32).contiguous() if ids.dtype != torch.int32 else ids.contiguous()
    raw = ctypes.c_void_p()
    torch.cuda.current_stream(pos.device).synchronize()
    _check(lib.bdm_slab_init(ctypes.byref(raw), n, capacity, _ptr(ids32), _ptr(pos.contiguous()),
                             _ptr(diam.contiguous()), ctypes.byref(p)))
    h = Handle(raw, n, True)
    h.capacity = capacity
    if stream is not None:
        bdm_set_stream(h, stream)
    return h


def bdm_slab_load(h: Handle, ids, pos, diam) -> None:
    """Replace the owned agents (CUDA tensors; ids as int32/int64)."""
    import torch

    ids32 = ids.to(torch.int32).contiguous() if ids.dtype != torch.int32 else ids.contiguous()
    _check(load_library().bdm_slab_load(h.raw, pos.shape[0], _ptr(ids32), _ptr(pos.contiguous()),
                                        _ptr(diam.contiguous())), h.raw)
    h.n = pos.shape[0]


def bdm_slab_local_maxd(h: Handle) -> float:
    v = ctypes.c_double(0.0)
    _check(load_library().bdm_slab_local_maxd(h.raw, ctypes.byref(v)), h.raw)
    return v.value


def bdm_slab_set_box_edge(h: Handle, L: float) -> None:
    _check(load_library().bdm_slab_set_box_edge(h.raw, float(L)), h.raw)


def bdm_slab_local_extents(h: Handle):
    out = np.zeros(6, np.int32)
    _check(load_library().bdm_slab_local_extents(h.raw, _ptr(out)), h.raw)
    return out[:3].copy(), out[3:].copy()


def bdm_slab_pack(h: Handle, what: int, x_begin: int, x_end: int, send_lo, send_hi, cap: int):
    """Returns (rc, n_lo, n_hi); rc is BDM_OK or BDM_ETRUNC (buffers too small, nothing committed)."""
    nlo, nhi = ctypes.c_int64(0), ctypes.c_int64(0)
    rc = load_library().bdm_slab_pack(h.raw, what, x_begin, x_end, _ptr(send_lo), _ptr(send_hi), cap,
                                      ctypes.byref(nlo), ctypes.byref(nhi))
    if rc not in (BDM_OK, BDM_ETRUNC):
        _check(rc, h.raw)
    return rc, nlo.value, nhi.value


def bdm_slab_split(h: Handle, x_begin: int, x_end: int, send_lo, send_hi, cap: int, info) -> None:
    """Asynchronous post-step split (emigrants front, halo back of send_*); counts into the DEVICE
    int64[12] tensor info."""
    _check(load_library().bdm_slab_split(h.raw, x_begin, x_end, _ptr(send_lo), _ptr(send_hi), cap, _ptr(info)),
           h.raw)


def bdm_slab_commit(h: Handle, n_stay: int) -> None:
    _check(load_library().bdm_slab_commit(h.raw, int(n_stay)), h.raw)


def bdm_slab_add(h: Handle, recv_lo, n_lo: int, recv_hi, n_hi: int) -> None:
    _check(load_library().bdm_slab_add(h.raw, _ptr(recv_lo) if n_lo else None, n_lo,
                                       _ptr(recv_hi) if n_hi else None, n_hi), h.raw)


def bdm_slab_step(h: Handle, glo3, ghi3, x_begin: int, x_end: int, recv_lo, n_lo: int, recv_hi, n_hi: int,
                  want_dp: bool = False) -> None:
    lo = np.ascontiguousarray(glo3, np.int32)
    hi = np.ascontiguousarray(ghi3, np.int32)
    _check(load_library().bdm_slab_step(h.raw, _ptr(lo), _ptr(hi), x_begin, x_end,
                                        _ptr(recv_lo) if n_lo else None, n_lo,
                                        _ptr(recv_hi) if n_hi else None, n_hi, int(want_dp)), h.raw)


def bdm_slab_get(h: Handle, what: int):
    """(ids int64 CUDA tensor, values [n,3] fp64 CUDA tensor) of the owned agents / last displacements."""
    import torch

    lib = load_library()
    n = ctypes.c_int64(0)
    _check(lib.bdm_slab_get(h.raw, what, ctypes.byref(n), None, None), h.raw)
    ids = torch.empty(n.value, dtype=torch.int32, device="cuda")
    vals = torch.empty((n.value, 3), dtype=torch.float64, device="cuda")
    _check(lib.bdm_slab_get(h.raw, what, ctypes.byref(n), _ptr(ids), _ptr(vals)), h.raw)
    return ids.to(torch.int64) & 0xFFFFFFFF, vals


# ------------------------------------------------------------------------------ distributed handles
def bdm_nccl_unique_id() -> bytes:
    """128-byte NCCL communicator id (rank 0 creates it and broadcasts it to the other ranks)."""
    buf = ctypes.create_string_buffer(128)
    _check(load_library().bdm_nccl_unique_id(buf))
    return buf.raw


def _dist_arrays(ids, pos, diam, p):
    dev = _is_torch(pos) and pos.is_cuda
    if dev:
        import torch

        assert pos.dtype == torch.float64 and diam.dtype == torch.float64 and ids.dtype == torch.int64
        assert pos.is_contiguous() and diam.is_contiguous() and ids.is_contiguous()
        p.flags |= BDM_DEVICE_PTRS
    else:
        p.flags &= ~BDM_DEVICE_PTRS
        pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
        diam = np.ascontiguousarray(diam, dtype=np.float64).reshape(-1)
        ids = np.ascontiguousarray(ids, dtype=np.int64).reshape(-1)
    if not (len(ids) == len(diam) == pos.shape[0]):
        raise ValueError("ids, pos and diam lengths differ")
    return ids, pos, diam, dev


def bdm_init_dist(ids, pos, diam, params: bdm_params | None = None, rank: int = 0, world: int = 1,
                  uid: bytes | None = None, device: int = 0, stream=None) -> Handle:
    """Collective: this rank's agents (global int64 ids, [n,3] positions, [n] diameters; NumPy or
    CUDA tensors) -> a distributed handle over `world` ranks (one process per GPU)."""
    p = params if params is not None else bdm_params_default()
    ids, pos, diam, dev = _dist_arrays(ids, pos, diam, p)
    p.device = device
    raw = ctypes.c_void_p()
    sp = getattr(stream, "cuda_stream", stream)
    if dev:
        import torch

        torch.cuda.synchronize(device)
    ubuf = ctypes.create_string_buffer(bytes(uid), 128)
    _check(load_library().bdm_init_dist(ctypes.byref(raw), len(diam), _ptr(ids), _ptr(pos), _ptr(diam),
                                        ctypes.byref(p), rank, world, ubuf, device, ctypes.c_void_p(sp or 0)))
    h = Handle(raw, 0, dev)
    h.world = world
    bdm_get_count(h)
    return h


def bdm_init_dist_local(world: int, counts, ids, pos, diam, params: bdm_params | None = None,
                        stream=None) -> Handle:
    """Virtual ranks (one GPU, one process): counts[r] agents of the concatenated arrays start on
    rank r; every exchange is a self send/recv of a 1-rank NCCL communicator."""
    p = params if params is not None else bdm_params_default()
    ids, pos, diam, dev = _dist_arrays(ids, pos, diam, p)
    c = np.ascontiguousarray(counts, dtype=np.int64)
    assert len(c) == world and int(c.sum()) == len(diam)
    if dev:
        import torch

        if p.device < 0:
            p.device = pos.device.index
        torch.cuda.synchronize()
    raw = ctypes.c_void_p()
    sp = getattr(stream, "cuda_stream", stream)
    _check(load_library().bdm_init_dist_local(ctypes.byref(raw), world, _ptr(c), _ptr(ids), _ptr(pos), _ptr(diam),
                                              ctypes.byref(p), ctypes.c_void_p(sp or 0)))
    h = Handle(raw, 0, dev)
    h.world = world
    bdm_get_count(h)
    return h


def bdm_set_agents_dist(h: Handle, ids, pos, diam) -> None:
    """Collective: a new batch for a distributed handle (redistributed; communicator and buffers reused)."""
    p = bdm_params()
    if h.device_ptrs:
        p.flags |= BDM_DEVICE_PTRS
    ids, pos, diam, dev = _dist_arrays(ids, pos, diam, p)
    if dev != h.device_ptrs:
        raise ValueError("host / device arrays must match the handle's mode")
    if dev:
        import torch

        torch.cuda.synchronize()
    _check(load_library().bdm_set_agents_dist(h.raw, len(diam), _ptr(ids), _ptr(pos), _ptr(diam)), h.raw)
    bdm_get_count(h)


def bdm_get_local(h: Handle, what: int = BDM_OWNED_POSITIONS):
    """(ids [n] int64, values [n,3]) of the owned agents of a distributed handle: positions or the
    displacements of the last step."""
    lib = load_library()
    n = ctypes.c_int64(0)
    _check(lib.bdm_get_local(h.raw, what, ctypes.byref(n), None, None), h.raw)
    m = int(n.value)
    if h.device_ptrs:
        import torch

        ids = torch.empty(m, dtype=torch.int64, device="cuda")
        vals = torch.empty((m, 3), dtype=torch.float64, device="cuda")
    else:
        ids = np.empty(m, np.int64)
        vals = np.empty((m, 3), np.float64)
    _check(lib.bdm_get_local(h.raw, what, ctypes.byref(n), _ptr(ids), _ptr(vals)), h.raw)
    return ids, vals


def bdm_get_cuts(h: Handle) -> list:
    out = np.zeros(h.world + 1, np.int32)
    _check(load_library().bdm_get_cuts(h.raw, _ptr(out), len(out)), h.raw)
    return [int(v) for v in out]


def bdm_get_pair_digest(h: Handle, kind: int):
    """(count [n] uint32, hash [n] uint64) of the neighbour (0) or contact (1) partners, id order."""
    n, _ = bdm_get_count(h)
    if h.device_ptrs:
        import torch

        cnt = torch.empty(n, dtype=torch.int32, device="cuda")
        hs = torch.empty(n, dtype=torch.int64, device="cuda")
    else:
        cnt = np.empty(n, np.uint32)
        hs = np.empty(n, np.uint64)
    _check(load_library().bdm_get_pair_digest(h.raw, kind, _ptr(cnt), _ptr(hs)), h.raw)
    return cnt, hs


def bdm_get_stats(h: Handle) -> dict:
    st = bdm_stats()
    _check(load_library().bdm_get_stats(h.raw, ctypes.byref(st)), h.raw)
    return {k: int(getattr(st, k)) for k, _ in bdm_stats._fields_}
