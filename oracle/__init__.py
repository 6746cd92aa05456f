"""CPU oracle for the BioDynaMo mechanical step -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import anything under oracle/.  The product package paper_2006_06775_b200 never imports it and
shares no code with it.

Two independent transcriptions of DESIGN.md §3 (O1-O8):
  * oracle/bdm_oracle.c  -- plain C grid oracle (qsort + binary search, -ffp-contract=off),
                            loaded here through ctypes as liboracle.so;
  * oracle/brute.py      -- O(N^2) NumPy brute force for tiny inputs.
Parity status of every function is listed in DESIGN.md §3.4 ("parity unpinned" items are named).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

_f64p = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)


class Params(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in
                ("k_rep", "gamma_att", "adherence", "dt", "eta", "max_disp", "box_edge_min")]


class Growth(ctypes.Structure):
    _fields_ = [("growth", ctypes.c_double), ("div_diam", ctypes.c_double), ("seed", ctypes.c_uint64)]


class Fields(ctypes.Structure):
    _fields_ = [("h", ctypes.c_double), ("origin", ctypes.c_double * 3), ("dims", ctypes.c_int32 * 3),
                ("diff", ctypes.c_double), ("decay", ctypes.c_double), ("dt", ctypes.c_double),
                ("secretion", ctypes.c_double), ("speed", ctypes.c_double)]


def fields(h, origin, dims, diff, decay, dt, secretion, speed) -> "Fields":
    return Fields(h, (ctypes.c_double * 3)(*origin), (ctypes.c_int32 * 3)(*dims), diff, decay, dt, secretion, speed)


class Grid(ctypes.Structure):
    _fields_ = [("L", ctypes.c_double), ("L2", ctypes.c_double), ("inv", ctypes.c_double),
                ("lo", ctypes.c_int64 * 3), ("hi", ctypes.c_int64 * 3)]


class Record(ctypes.Structure):
    _fields_ = [("n_cand", ctypes.c_void_p), ("n_nb", ctypes.c_void_p), ("n_ct", ctypes.c_void_p),
                ("s_abs", ctypes.c_void_p), ("branch", ctypes.c_void_p), ("nb_hash", ctypes.c_void_p),
                ("ct_hash", ctypes.c_void_p), ("force", ctypes.c_void_p)]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc -O2 -ffp-contract=off -fopenmp (building is not using it)."""
    src = os.path.join(HERE, "bdm_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
                               "-shared", "-o", LIB_PATH, src, "-lm"])
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        L.orc_grid_params.argtypes = [ctypes.c_int64, _f64p, _f64p, ctypes.c_double, ctypes.POINTER(Grid)]
        L.orc_step_sample.argtypes = [ctypes.c_int64, _f64p, _f64p, ctypes.POINTER(Params), ctypes.c_int64, _i64p,
                                      _f64p, _f64p, ctypes.POINTER(Record), ctypes.c_int]
        L.orc_step.argtypes = [ctypes.c_int64, _f64p, _f64p, ctypes.POINTER(Params), _f64p, _f64p,
                               ctypes.POINTER(Record), ctypes.c_int]
        L.orc_run.argtypes = [ctypes.c_int64, _f64p, _f64p, ctypes.POINTER(Params), ctypes.c_int32, _f64p,
                              ctypes.c_int]
        L.orc_pairs.argtypes = [ctypes.c_int64, _f64p, _f64p, ctypes.POINTER(Params), ctypes.c_int, _i64p,
                                ctypes.c_int64]
        L.orc_pairs.restype = ctypes.c_int64
        L.orc_pair_force.argtypes = [_f64p, _f64p, ctypes.c_double, ctypes.c_double, ctypes.c_int64,
                                     ctypes.c_int64, ctypes.POINTER(Params), _f64p]
        L.orc_displacement.argtypes = [_f64p, ctypes.POINTER(Params), _f64p]
        L.orc_box_coords.argtypes = [ctypes.c_int64, _f64p, ctypes.POINTER(Grid), _i64p]
        L.orc_grow_divide.argtypes = [ctypes.c_int64, _f64p, _f64p, ctypes.POINTER(Growth), ctypes.c_int64,
                                      ctypes.c_int64]
        L.orc_grow_divide.restype = ctypes.c_int64
        L.orc_run_growth.argtypes = [ctypes.c_int64, _f64p, _f64p, ctypes.POINTER(Params), ctypes.POINTER(Growth),
                                     ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, _f64p, ctypes.c_int]
        L.orc_run_growth.restype = ctypes.c_int64
        _i8p = ctypes.POINTER(ctypes.c_int8)
        L.orc_secrete.argtypes = [ctypes.c_int64, _f64p, _i8p, ctypes.POINTER(Fields), _f64p, _f64p]
        L.orc_diffuse.argtypes = [ctypes.POINTER(Fields), _f64p, _f64p]
        L.orc_gradient_at.argtypes = [ctypes.POINTER(Fields), _f64p, _f64p, _f64p]
        L.orc_chemotaxis.argtypes = [ctypes.c_int64, _f64p, _i8p, ctypes.POINTER(Fields), _f64p, _f64p]
        L.orc_run_soma.argtypes = [ctypes.c_int64, _f64p, _f64p, _i8p, ctypes.POINTER(Params), ctypes.POINTER(Fields),
                                   _f64p, _f64p, ctypes.c_int32, _f64p, ctypes.c_int]
        L.orc_neurite_step.argtypes = [ctypes.c_int64, _f64p, _f64p, ctypes.c_int64, _f64p, _f64p, _f64p, _f64p,
                                       _i64p, _i64p, _i64p, ctypes.POINTER(Params), ctypes.POINTER(ctypes.c_double),
                                       _f64p, _f64p]
        L.orc_mix64.argtypes = [ctypes.c_uint64]
        L.orc_mix64.restype = ctypes.c_uint64
        _lib = L
    return _lib


DEFAULTS = dict(k_rep=10.0, gamma_att=4.0, adherence=0.1, dt=1.0, eta=1.0, max_disp=3.0, box_edge_min=0.0)


def params(**kw) -> Params:
    d = dict(DEFAULTS)
    d.update(kw)
    return Params(**d)


def _ptr(a, t=_f64p):
    return a.ctypes.data_as(t)


def _c(a, dtype=np.float64):
    return np.ascontiguousarray(a, dtype=dtype)


def grid_params(pos, diam, box_edge_min=0.0):
    pos, diam = _c(pos), _c(diam)
    g = Grid()
    rc = lib().orc_grid_params(len(diam), _ptr(pos), _ptr(diam), box_edge_min, ctypes.byref(g))
    if rc:
        raise OracleError(rc)
    return dict(L=g.L, L2=g.L2, inv=g.inv, lo=tuple(g.lo), hi=tuple(g.hi))


def box_coords(pos, diam, box_edge_min=0.0):
    """O2: integer box coordinates of every agent under the grid of O1."""
    pos, diam = _c(pos), _c(diam)
    g = Grid()
    rc = lib().orc_grid_params(len(diam), _ptr(pos), _ptr(diam), box_edge_min, ctypes.byref(g))
    if rc:
        raise OracleError(rc)
    b = np.zeros((len(diam), 3), np.int64)
    lib().orc_box_coords(len(diam), _ptr(pos), ctypes.byref(g), _ptr(b, _i64p))
    return b


class OracleError(RuntimeError):
    def __init__(self, rc):
        super().__init__(f"oracle error {rc}")
        self.rc = rc


def step(pos, diam, prm=None, sample=None, record=True, nthreads=0):
    """One step O1-O7.  Returns dict(dp, pos_new, and per-agent records indexed by id)."""
    pos, diam = _c(pos), _c(diam)
    n = len(diam)
    prm = prm or params()
    m = n if sample is None else len(sample)
    dp = np.zeros((m, 3))
    pn = np.zeros((m, 3))
    out = dict(dp=dp, pos_new=pn)
    rec = None
    if record:
        out.update(n_cand=np.zeros(n, np.int32), n_nb=np.zeros(n, np.int32), n_ct=np.zeros(n, np.int32),
                   s_abs=np.zeros(n), branch=np.full(n, -1, np.int8), nb_hash=np.zeros(n, np.uint64),
                   ct_hash=np.zeros(n, np.uint64), force=np.zeros((n, 3)))
        rec = Record(*(out[k].ctypes.data for k in
                       ("n_cand", "n_nb", "n_ct", "s_abs", "branch", "nb_hash", "ct_hash", "force")))
    smp = None
    if sample is not None:
        smp = _c(sample, np.int64)
    rc = lib().orc_step_sample(n, _ptr(pos), _ptr(diam), ctypes.byref(prm), m,
                               _ptr(smp, _i64p) if smp is not None else None, _ptr(dp), _ptr(pn),
                               ctypes.byref(rec) if rec is not None else None, nthreads)
    if rc:
        raise OracleError(rc)
    return out


def run(pos, diam, n_steps, prm=None, nthreads=0):
    pos, diam = _c(pos).copy(), _c(diam)
    dp = np.zeros_like(pos)
    rc = lib().orc_run(len(diam), _ptr(pos), _ptr(diam), ctypes.byref(prm or params()), n_steps, _ptr(dp),
                       nthreads)
    if rc:
        raise OracleError(rc)
    return pos, dp


def pairs(pos, diam, kind, prm=None):
    """kind 0: neighbour set N; kind 1: contact set C.  Sorted (i<j) int64 [P,2]."""
    pos, diam = _c(pos), _c(diam)
    prm = prm or params()
    cap = 0
    while True:
        out = np.zeros((max(cap, 1), 2), np.int64)
        cnt = lib().orc_pairs(len(diam), _ptr(pos), _ptr(diam), ctypes.byref(prm), kind, _ptr(out, _i64p), cap)
        if cnt < 0:
            raise OracleError(cnt)
        if cnt <= cap:
            return out[:cnt]
        cap = cnt


def pair_force(pi, pj, Di, Dj, idi=0, idj=1, prm=None):
    pi, pj = _c(pi), _c(pj)
    t = np.zeros(3)
    c = lib().orc_pair_force(_ptr(pi), _ptr(pj), Di, Dj, idi, idj, ctypes.byref(prm or params()), _ptr(t))
    return bool(c), t


def displacement(F, prm=None):
    F = _c(F)
    dp = np.zeros(3)
    br = lib().orc_displacement(_ptr(F), ctypes.byref(prm or params()), _ptr(dp))
    return dp, br


def mix64(x: int) -> int:
    return int(lib().orc_mix64(x))


def threads() -> int:
    return int(lib().orc_threads())


def grow_divide(pos, diam, growth, div_diam, seed, step):
    """NEXT-2 G1-G2 on copies; returns (pos, diam) with daughters appended (ids n, n+1, ...)."""
    n = len(diam)
    cap = 2 * n + 1
    P = np.zeros((cap, 3))
    Dm = np.zeros(cap)
    P[:n] = pos
    Dm[:n] = diam
    m = lib().orc_grow_divide(n, _ptr(P), _ptr(Dm), ctypes.byref(Growth(growth, div_diam, seed)), step, cap)
    if m < 0:
        raise OracleError(m)
    return P[:m].copy(), Dm[:m].copy()


def run_growth(pos, diam, n_steps, growth, div_diam, seed, prm=None, step0=0, cap=None):
    """n_steps of (mechanics, growth + division).  Returns (pos, diam, dp of the last mechanics)."""
    n = len(diam)
    cap = cap or max(4 * n, 16) * (2 ** min(n_steps, 6))
    P = np.zeros((cap, 3))
    Dm = np.zeros(cap)
    P[:n] = pos
    Dm[:n] = diam
    dp = np.zeros((cap, 3))
    m = lib().orc_run_growth(n, _ptr(P), _ptr(Dm), ctypes.byref(prm or params()),
                             ctypes.byref(Growth(growth, div_diam, seed)), n_steps, step0, cap, _ptr(dp), 0)
    if m < 0:
        raise OracleError(m)
    return P[:m].copy(), Dm[:m].copy(), dp


_i8p = ctypes.POINTER(ctypes.c_int8)


def diffuse(fp, c):
    """S2 on a copy of field c (shape dims)."""
    c = _c(c)
    out = np.zeros_like(c)
    lib().orc_diffuse(ctypes.byref(fp), _ptr(c), _ptr(out))
    return out


def secrete(fp, pos, types, c0, c1):
    pos = _c(pos)
    t = _c(types, np.int8)
    c0, c1 = _c(c0).copy(), _c(c1).copy()
    lib().orc_secrete(len(t), _ptr(pos), _ptr(t, _i8p), ctypes.byref(fp), _ptr(c0), _ptr(c1))
    return c0, c1


def gradient_at(fp, c, p):
    c, p = _c(c), _c(p)
    g = np.zeros(3)
    lib().orc_gradient_at(ctypes.byref(fp), _ptr(c), _ptr(p), _ptr(g))
    return g


def run_soma(pos, diam, types, fp, n_steps, c0=None, c1=None, prm=None):
    """n_steps of S1-S4.  Returns (pos, c0, c1, dp of the last mechanics)."""
    pos, diam = _c(pos).copy(), _c(diam)
    t = _c(types, np.int8)
    dims = tuple(fp.dims)
    c0 = np.zeros(dims) if c0 is None else _c(c0).copy()
    c1 = np.zeros(dims) if c1 is None else _c(c1).copy()
    dp = np.zeros_like(pos)
    rc = lib().orc_run_soma(len(diam), _ptr(pos), _ptr(diam), _ptr(t, _i8p), ctypes.byref(prm or params()),
                            ctypes.byref(fp), _ptr(c0), _ptr(c1), n_steps, _ptr(dp), 0)
    if rc:
        raise OracleError(rc)
    return pos, c0, c1, dp


def neurite_step(pos, diam, Q, de, l0, anchor, mother, c1, c2, k_spring, prm=None, steps=1):
    """NEXT-4 (N1-N6): spheres + neurite elements, `steps` Jacobi steps.  Returns (pos, Q, dp, dQ)."""
    pos, diam = _c(pos).copy(), _c(diam)
    Q, de, l0, A = _c(Q).copy(), _c(de), _c(l0), _c(anchor)
    m, a1, a2 = _c(mother, np.int64), _c(c1, np.int64), _c(c2, np.int64)
    dp = np.zeros_like(pos)
    dQ = np.zeros_like(Q)
    ks = ctypes.c_double(k_spring)
    for _ in range(steps):
        rc = lib().orc_neurite_step(len(diam), _ptr(pos), _ptr(diam), len(de), _ptr(Q), _ptr(de), _ptr(l0), _ptr(A),
                                    _ptr(m, _i64p), _ptr(a1, _i64p), _ptr(a2, _i64p), ctypes.byref(prm or params()),
                                    ctypes.byref(ks), _ptr(dp), _ptr(dQ))
        if rc:
            raise OracleError(rc)
    return pos, Q, dp, dQ
