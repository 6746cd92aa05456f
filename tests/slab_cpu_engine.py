"""Test double of dist.GpuSlabEngine for the CPU tests of the x-slab protocol.

It keeps a rank's owned agents in NumPy and computes a step with the CPU oracle over owned + ghost
agents (the oracle is test infrastructure; this engine never runs outside tests/).  Agents are
ordered by global id before calling the oracle so that its index order is the global id order
(canonical in-box order, coincident tie-break), and box_edge_min = the global L so that the oracle
bins with the same box edge as the single-process run.  With a correct protocol, the positions
after K slab steps equal the single-process oracle's bit for bit.
"""
import numpy as np
import torch

import oracle

INT32_MIN = -(2 ** 31)
INT32_MAX = 2 ** 31 - 1


class CpuSlabEngine:
    def __init__(self, ids, pos, diam, prm=None):
        self.ids = np.asarray(ids, np.int64)
        self.pos = np.asarray(pos, np.float64).reshape(-1, 3).copy()
        self.diam = np.asarray(diam, np.float64).copy()
        self.prm = dict(oracle.DEFAULTS, **(prm or {}))
        self.ext = None
        self.last = None

    def local_maxd(self):
        return float(self.diam.max()) if len(self.diam) else 0.0

    def max_disp(self):
        return float(self.prm["max_disp"])

    def box_edge_min(self):
        return float(self.prm["box_edge_min"])

    def set_box_edge(self, L):
        self.L = max(L, self.prm["box_edge_min"])
        self.inv = 1.0 / (self.L * (1.0 + 2.0 ** -30))
        self.ext = None

    def _bx(self):
        return np.floor(self.pos[:, 0] * self.inv).astype(np.int64)

    def local_extents(self):
        if self.ext is None:
            if len(self.ids) == 0:
                self.ext = (np.full(3, INT32_MAX), np.full(3, INT32_MIN))
            else:
                b = np.floor(self.pos * self.inv).astype(np.int64)
                self.ext = (b.min(0), b.max(0))
        return self.ext

    def _rec(self, m):
        return torch.from_numpy(np.concatenate([self.pos[m], self.diam[m, None], self.ids[m, None].astype(np.float64)],
                                               axis=1).reshape(-1, 5).copy())

    def pack(self, what, xb, xe):
        bx = self._bx()
        if what == 0:
            lo = (bx == xb) & (xb != INT32_MIN)
            hi = (bx == xe - 1) & (xe != INT32_MAX)
            return self._rec(lo), self._rec(hi)
        lo, hi = bx < xb, bx >= xe
        out = self._rec(lo), self._rec(hi)
        keep = ~(lo | hi)
        self.ids, self.pos, self.diam = self.ids[keep], self.pos[keep], self.diam[keep]
        return out

    def split(self, xb, xe):
        """Single-sync protocol: emigrants at the front, boundary stayers at the back of each buffer
        (cap = owned count); counts and extents in info (as bdm_slab_split)."""
        bx = self._bx()
        mlo, mhi = bx < xb, bx >= xe
        keep = ~(mlo | mhi)
        hlo = keep & (bx == xb) & (xb != INT32_MIN)
        hhi = keep & (bx == xe - 1) & (xe != INT32_MAX)
        cap = max(len(self.ids), 1)
        bufs = []
        for m, h in ((mlo, hlo), (mhi, hhi)):
            b = torch.zeros((cap, 5), dtype=torch.float64)
            nm, nh = int(m.sum()), int(h.sum())
            b[:nm] = self._rec(m)
            if nh:
                b[cap - nh:] = torch.flip(self._rec(h), dims=[0])
            bufs.append(b)
        lo, hi = self.local_extents()
        info = torch.tensor([int(mlo.sum()), int(hlo.sum()), int(mhi.sum()), int(hhi.sum()), int(keep.sum()),
                             *[int(v) for v in lo], *[int(v) for v in hi], 0], dtype=torch.int64)
        self.pending = keep
        return bufs[0], bufs[1], info

    def commit(self, n_stay):
        keep, self.pending = self.pending, None
        if n_stay < 0:
            return
        assert int(keep.sum()) == n_stay
        self.ids, self.pos, self.diam = self.ids[keep], self.pos[keep], self.diam[keep]
        self.ext = None

    def grow_buffers(self, need):
        pass

    def add(self, rl, rh):
        for r in (rl, rh):
            r = r.numpy()
            if len(r):
                self.ext = None
                self.pos = np.concatenate([self.pos, r[:, :3]])
                self.diam = np.concatenate([self.diam, r[:, 3]])
                self.ids = np.concatenate([self.ids, r[:, 4].astype(np.int64)])

    def step(self, glo, ghi, xb, xe, gl, gh, want_dp=False):
        g = np.concatenate([gl.numpy(), gh.numpy()]).reshape(-1, 5)
        gb = np.floor(g[:, 0] * self.inv).astype(np.int64)
        assert np.all((gb == xb - 1) | (gb == xe)), "ghost outside the halo layers"
        assert np.all((self._bx() >= xb) & (self._bx() < xe)), "owned agent outside the slab"
        ids = np.concatenate([self.ids, g[:, 4].astype(np.int64)])
        pos = np.concatenate([self.pos, g[:, :3]])
        diam = np.concatenate([self.diam, g[:, 3]])
        order = np.argsort(ids, kind="stable")
        own = np.flatnonzero(order < len(self.ids))  # positions (in id order) of owned agents
        p = dict(self.prm, box_edge_min=self.L)
        r = oracle.step(pos[order], diam[order], oracle.params(**p), sample=own, record=False)
        src = order[own]  # index into owned arrays
        self.pos[src] = r["pos_new"]
        self.last = (self.ids[src].copy(), r["dp"])
        b = np.floor(self.pos * self.inv).astype(np.int64) if len(self.ids) else None
        self.ext = (b.min(0), b.max(0)) if b is not None else (np.full(3, INT32_MAX), np.full(3, INT32_MIN))

    def owned(self):
        return self.ids.copy(), self.pos.copy()
