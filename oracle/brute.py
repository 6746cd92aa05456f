"""O(N^2) brute-force oracle (NumPy, fp64) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import this.
It is a second, independent transcription of DESIGN.md §3 O1-O7 that does
not use a grid at all: every pair i<j is examined.  It is the pin for the grid oracle's
neighbour search (§2.1: the 27-box search must find every interaction
because the box edge is the largest diameter) and is only meant for N <= a few thousand.

NumPy elementwise ops on float64 are separately rounded IEEE operations (no FMA), matching
O3/O4 term by term.  Sums run in ascending j (pure-Python loop over each agent's contacts).
"""
from __future__ import annotations

import math

import numpy as np

DEFAULTS = dict(k_rep=10.0, gamma_att=4.0, adherence=0.1, dt=1.0, eta=1.0, max_disp=3.0, box_edge_min=0.0)


def grid_params(diam, box_edge_min=0.0):
    """O1: box edge L, L2, binning inverse."""
    L = max(float(np.max(diam)) if len(diam) else 0.0, box_edge_min)
    return L, L * L, 1.0 / (L * (1.0 + 2.0 ** -30))


def box_coords(pos, inv):
    """O2: integer box coordinates floor(p * inv)."""
    return np.floor(pos * inv).astype(np.int64)


def all_pairs(pos, diam, params=None):
    """Neighbour set N (d2 <= L2) and contact set C (delta > 0) as sorted (i<j) int64 arrays.

    Also returns, per contact pair, the force on the lower id (O4)."""
    p = dict(DEFAULTS, **(params or {}))
    n = len(diam)
    L, L2, _ = grid_params(diam, p["box_edge_min"])
    nb, ct, ctf = [], [], []
    for i in range(n - 1):
        j = np.arange(i + 1, n)
        dx = pos[i, 0] - pos[j, 0]
        dy = pos[i, 1] - pos[j, 1]
        dz = pos[i, 2] - pos[j, 2]
        d2 = (dx * dx + dy * dy) + dz * dz
        m = d2 <= L2
        for jj, ddx, ddy, ddz, dd2 in zip(j[m], dx[m], dy[m], dz[m], d2[m]):
            nb.append((i, jj))
            t = _pair(float(ddx), float(ddy), float(ddz), float(dd2), diam[i], diam[jj], i, int(jj), p)
            if t is not None:
                ct.append((i, jj))
                ctf.append(t)
    nb = np.array(nb, dtype=np.int64).reshape(-1, 2)
    ct = np.array(ct, dtype=np.int64).reshape(-1, 2)
    return nb, ct, ctf


def _pair(dx, dy, dz, d2, Di, Dj, idi, idj, p):
    """O4 for one pair; returns (force on i, |f|) or None when delta <= 0."""
    d = math.sqrt(d2)
    ri = 0.5 * float(Di)
    rj = 0.5 * float(Dj)
    s = ri + rj
    delta = s - d
    if not delta > 0.0:
        return None
    r = (ri * rj) / s
    f = p["k_rep"] * delta - p["gamma_att"] * math.sqrt(r * delta)
    if d2 == 0.0:
        sign = 1.0 if idi > idj else -1.0
        return (sign * f, 0.0, 0.0), abs(f)
    m = f / d
    return (m * dx, m * dy, m * dz), abs(f)


def displacement(F, p):
    """O6 (north_star adherence threshold + max-displacement clamp)."""
    fn = math.sqrt((F[0] * F[0] + F[1] * F[1]) + F[2] * F[2])
    if fn <= p["adherence"]:
        return (0.0, 0.0, 0.0), 0
    c = p["dt"] / p["eta"]
    if fn * c > p["max_disp"]:
        scale = p["max_disp"] / fn
        return (F[0] * scale, F[1] * scale, F[2] * scale), 1
    return (F[0] * c, F[1] * c, F[2] * c), 2


def step(pos, diam, params=None):
    """O1-O7 by brute force.  Returns dict with dp, pos_new, force, branch, n_nb, n_ct, s_abs."""
    p = dict(DEFAULTS, **(params or {}))
    pos = np.ascontiguousarray(pos, dtype=np.float64)
    diam = np.ascontiguousarray(diam, dtype=np.float64)
    n = len(diam)
    nb, ct, ctf = all_pairs(pos, diam, p)
    terms = [[] for _ in range(n)]  # (j, term on i)
    s_abs = np.zeros(n)
    for (i, j), (t, fa) in zip(ct, ctf):
        terms[i].append((j, t))
        terms[j].append((i, (-t[0], -t[1], -t[2])))
        s_abs[i] += fa
        s_abs[j] += fa
    F = np.zeros((n, 3))
    dp = np.zeros((n, 3))
    branch = np.zeros(n, dtype=np.int8)
    for i in range(n):
        fx = fy = fz = 0.0
        for _, t in sorted(terms[i], key=lambda e: e[0]):  # ascending j
            fx = fx + t[0]
            fy = fy + t[1]
            fz = fz + t[2]
        F[i] = (fx, fy, fz)
        dp[i], branch[i] = displacement((fx, fy, fz), p)
    n_nb = np.bincount(nb.ravel(), minlength=n).astype(np.int32) if n else np.zeros(0, np.int32)
    n_ct = np.bincount(ct.ravel(), minlength=n).astype(np.int32) if n else np.zeros(0, np.int32)
    return dict(dp=dp, pos_new=pos + dp, force=F, branch=branch, n_nb=n_nb, n_ct=n_ct, s_abs=s_abs, nb=nb, ct=ct)
