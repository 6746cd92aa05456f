"""Reference model of the x-slab protocol -- TEST INFRASTRUCTURE.

The product path is libbdm.so's distributed runtime (bdm_init_dist, csrc/bdm_dist.cuh), which owns
the exchange's data plane (NCCL) and runs it with device-resident counts.  This module is the same
protocol written as host orchestration over the slab building blocks of the C ABI (bdm_slab_*), so
that it can run against a CPU oracle engine over gloo (tests/test_slabs_cpu.py) and against the
GPU kernels with in-process virtual slabs (tests/test_gpu_slabs.py).


north_star: "Across the 8 GPUs of one box the domain is split into x-slabs.  Each step does a halo
exchange of boundary-box agents and migrates agents that cross slab boundaries, using NCCL
send/recv over NVLink."

Rank g owns the agents whose integer box-x lies in [bounds[g], bounds[g+1]) (bounds[0] = INT32_MIN,
bounds[G] = INT32_MAX).  One step of the single-sync protocol (every slab at least 2 boxes wide):
  1. bdm_slab_step with the ghosts prepared by the previous step: slab-local grid over owned +
     ghosts, force / displacement / update of the owned agents (libbdm.so kernels);
  2. bdm_slab_split (device, no host round trip): emigrants (new box-x outside the slab) and the
     stayers of the first / last box-x layer (the neighbours' next ghosts) into the send buffers;
  3. on the device: counts to g-1 / g+1 and an allreduce of the box extents; then ONE host read of
     all counts and extents;
  4. payloads to g-1 / g+1; commit the stayers, append the immigrants; the next step's ghosts of a
     side are the neighbour's boundary stayers plus this rank's own emigrants to that side (they
     moved less than a box, so they sit exactly in the neighbour's boundary layer).
The legacy protocol (extents allreduce, halo pack + exchange, step, migration pack + exchange: six
host round trips) remains for slabs one box wide and for the setup.  Counts travel before payloads;
records are 5 fp64 (x, y, z, D, id).  The arithmetic is unchanged
from the single-GPU path and ghosts keep their global ids, so every owned agent's force is summed
in the same canonical order: results are bit-identical to one GPU.

This module is orchestration only (which buffer goes to which rank).  It runs against any engine
with the interface of GpuSlabEngine and any communicator with the interface of TorchComm -- the
CPU tests drive it with a gloo communicator and a test engine, the virtual-slab GPU test with
LoopComm (several slabs in one process).
"""
from __future__ import annotations

import json
import time

import os

import numpy as np

INT32_MIN = -(2 ** 31)
INT32_MAX = 2 ** 31 - 1
REC = 5


def choose_bounds(hist: np.ndarray, x0: int, world: int, weights: np.ndarray | None = None) -> list[int]:
    """Slab bounds on integer box-x from a global histogram (hist[k] = agents with box-x = x0 + k).

    Cuts balance the (optionally weighted) agent count; every slab is at least one box wide."""
    w = hist.astype(np.float64) if weights is None else weights.astype(np.float64)
    nx = len(w)
    bounds = [INT32_MIN]
    if world > 1:
        cum = np.cumsum(w)
        total = cum[-1] if nx else 0.0
        # inner slabs at least 2 boxes wide when the population spans enough boxes (the single-sync
        # protocol needs it), else 1
        wmin = 2 if nx >= 2 * world else 1
        prev = x0
        for g in range(1, world):
            target = total * g / world
            k = int(np.searchsorted(cum, target, side="left")) + 1  # first box of slab g (relative)
            cut = x0 + k
            cut = max(cut, prev + (1 if g == 1 else wmin))
            if nx >= world:
                cut = min(cut, x0 + nx - 1 - (world - 1 - g) * wmin)
            bounds.append(int(cut))
            prev = cut
    bounds.append(INT32_MAX)
    return bounds


# --------------------------------------------------------------------------------- communicators
class TorchComm:
    """One slab per process; exchange with ranks g-1 / g+1 over torch.distributed (NCCL or gloo)."""

    def __init__(self, device=None):
        import torch.distributed as dist

        self.dist = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.device = device

    def slab_ids(self):
        return [self.rank]

    def _t(self, arr, dtype):
        import torch

        return torch.as_tensor(np.asarray(arr), dtype=dtype, device=self.device)

    def allreduce_max(self, vals):
        import torch

        t = self._t([max(vals)], torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def allreduce_sum(self, arrs):
        import torch

        t = self._t(np.sum(np.stack(arrs), axis=0), torch.int64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return t.cpu().numpy()

    def allreduce_extents(self, exts):
        import torch

        (lo, hi), = exts
        t = self._t(np.concatenate([np.asarray(lo, np.int64), -np.asarray(hi, np.int64)]), torch.int64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN)
        v = t.cpu().numpy()
        return v[:3].astype(np.int64), (-v[3:]).astype(np.int64)

    def exchange(self, sends):
        """sends = [(to_lower, to_upper)] ([m,5] fp64 tensors); returns [(from_lower, from_upper)]."""
        import torch

        dist = self.dist
        (s_lo, s_hi), = sends
        r, G = self.rank, self.world
        dev = s_lo.device
        peers = [(r - 1, s_lo), (r + 1, s_hi)]
        cnt_out = {p: torch.tensor([t.shape[0]], dtype=torch.int64, device=dev) for p, t in peers if 0 <= p < G}
        cnt_in = {p: torch.zeros(1, dtype=torch.int64, device=dev) for p, _ in peers if 0 <= p < G}
        for p, t in peers:
            if not (0 <= p < G):
                assert t.shape[0] == 0, "records addressed to a rank outside the job"
        ops = []
        for p in cnt_out:
            ops.append(dist.P2POp(dist.isend, cnt_out[p], p))
            ops.append(dist.P2POp(dist.irecv, cnt_in[p], p))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        recv = {}
        ops = []
        for p, t in peers:
            if not (0 <= p < G):
                recv[p] = torch.empty((0, REC), dtype=torch.float64, device=dev)
                continue
            m = int(cnt_in[p].item())
            recv[p] = torch.empty((m, REC), dtype=torch.float64, device=dev)
            if t.shape[0]:
                ops.append(dist.P2POp(dist.isend, t.contiguous(), p))
            if m:
                ops.append(dist.P2POp(dist.irecv, recv[p], p))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        return [(recv[r - 1], recv[r + 1])]

    def exchange_split(self, splits):
        return _TorchSplitExchange.run(self, splits)


def _split_counts(info):
    """Host view of one slab's split info (int64[12]) -> dict."""
    return dict(mig_lo=int(info[0]), halo_lo=int(info[1]), mig_hi=int(info[2]), halo_hi=int(info[3]),
                n_stay=int(info[4]), lo=np.asarray(info[5:8], np.int64), hi=np.asarray(info[8:11], np.int64),
                overflow=int(info[11]))


class _TorchSplitExchange:
    """TorchComm.exchange_split (single-sync protocol step 3-4), NCCL or gloo."""

    @staticmethod
    def run(comm, splits):
        import torch

        dist = comm.dist
        (s_lo, s_hi, info), = splits
        r, G = comm.rank, comm.world
        dev = info.device
        cap = s_lo.shape[0]
        rc_lo = torch.zeros(2, dtype=torch.int64, device=dev)
        rc_hi = torch.zeros(2, dtype=torch.int64, device=dev)
        ops = []
        if r - 1 >= 0:
            ops += [dist.P2POp(dist.isend, info[0:2].contiguous(), r - 1), dist.P2POp(dist.irecv, rc_lo, r - 1)]
        if r + 1 < G:
            ops += [dist.P2POp(dist.isend, info[2:4].contiguous(), r + 1), dist.P2POp(dist.irecv, rc_hi, r + 1)]
        # extents (min lo, max hi) and any overflow, reduced with one MIN
        red = torch.cat([info[5:8], -info[8:11], -info[11:12]])
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        dist.all_reduce(red, op=dist.ReduceOp.MIN)
        host = torch.cat([info, rc_lo, rc_hi, red]).cpu().numpy()  # the step's one host round trip
        mine = _split_counts(host[:12])
        in_lo, in_hi = host[12:14], host[14:16]
        glo, ghi, any_overflow = host[16:19], -host[19:22], -host[22]
        out = dict(mine, glo=glo.astype(np.int64), ghi=ghi.astype(np.int64), any_overflow=int(any_overflow))
        if any_overflow:
            return [out]
        recv = {}
        ops = []
        for side, peer, buf, mig, halo, rin in (("lo", r - 1, s_lo, mine["mig_lo"], mine["halo_lo"], in_lo),
                                                ("hi", r + 1, s_hi, mine["mig_hi"], mine["halo_hi"], in_hi)):
            imm = torch.empty((int(rin[0]), REC), dtype=torch.float64, device=dev)
            hal = torch.empty((int(rin[1]), REC), dtype=torch.float64, device=dev)
            recv[side] = (imm, hal)
            if not (0 <= peer < G):
                assert mig == 0 and halo == 0, "records addressed to a rank outside the job"
                continue
            if mig:
                ops.append(dist.P2POp(dist.isend, buf[:mig], peer))
            if halo:
                ops.append(dist.P2POp(dist.isend, buf[cap - halo:], peer))
            if imm.shape[0]:
                ops.append(dist.P2POp(dist.irecv, imm, peer))
            if hal.shape[0]:
                ops.append(dist.P2POp(dist.irecv, hal, peer))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        out.update(imm_lo=recv["lo"][0], halo_in_lo=recv["lo"][1], imm_hi=recv["hi"][0], halo_in_hi=recv["hi"][1])
        return [out]


class LoopComm:
    """All slabs in one process: exchanges are hand-overs between the local slabs (virtual slabs on
    one GPU, or one CPU process).  Same interface as TorchComm with lists over all slabs."""

    def __init__(self, world: int):
        self.world = world

    def slab_ids(self):
        return list(range(self.world))

    def allreduce_max(self, vals):
        return float(max(vals))

    def allreduce_sum(self, arrs):
        return np.sum(np.stack(arrs), axis=0)

    def allreduce_extents(self, exts):
        lo = np.min(np.stack([np.asarray(e[0], np.int64) for e in exts]), axis=0)
        hi = np.max(np.stack([np.asarray(e[1], np.int64) for e in exts]), axis=0)
        return lo, hi

    def exchange(self, sends):
        G = self.world
        out = []
        for g in range(G):
            frm_lo = sends[g - 1][1] if g > 0 else sends[g][0][:0]
            frm_hi = sends[g + 1][0] if g + 1 < G else sends[g][1][:0]
            out.append((frm_lo, frm_hi))
        assert sends[0][0].shape[0] == 0 and sends[G - 1][1].shape[0] == 0
        return out

    def exchange_split(self, splits):
        G = self.world
        infos = [_split_counts(np.asarray(info.cpu().numpy())) for _, _, info in splits]
        glo = np.min(np.stack([c["lo"] for c in infos]), axis=0)
        ghi = np.max(np.stack([c["hi"] for c in infos]), axis=0)
        anyo = max(c["overflow"] for c in infos)
        outs = []
        for g in range(G):
            o = dict(infos[g], glo=glo, ghi=ghi, any_overflow=anyo)
            if not anyo:
                for side, nb, key_m, key_h in (("lo", g - 1, "mig_hi", "halo_hi"), ("hi", g + 1, "mig_lo", "halo_lo")):
                    if 0 <= nb < G:
                        buf = splits[nb][1] if side == "lo" else splits[nb][0]
                        cap = buf.shape[0]
                        m, hh = infos[nb][key_m], infos[nb][key_h]
                        o["imm_" + side], o["halo_in_" + side] = buf[:m], buf[cap - hh:]
                    else:
                        empty = splits[g][0][:0]
                        o["imm_" + side], o["halo_in_" + side] = empty, empty
            outs.append(o)
        assert infos[0]["mig_lo"] == infos[0]["halo_lo"] == 0 and infos[G - 1]["mig_hi"] == infos[G - 1]["halo_hi"] == 0
        return outs


# --------------------------------------------------------------------------------- GPU engine
class GpuSlabEngine:
    """One rank's slab on a GPU, through the C ABI (libbdm.so bdm_slab_*)."""

    def __init__(self, ids, pos, diam, capacity: int, params=None, device=None, stream=None):
        import torch

        import paper_2006_06775_b200 as bdm

        self.bdm = bdm
        self.torch = torch
        self.device = device if device is not None else pos.device
        self.params = params if params is not None else bdm.bdm_params_default()
        self.h = bdm.bdm_slab_init(ids, pos, diam, capacity, self.params, stream=stream)
        self.buf_cap = max(1024, capacity // 16)
        self._alloc()

    def _alloc(self):
        t = self.torch
        self.s_lo = t.empty((self.buf_cap, REC), dtype=t.float64, device=self.device)
        self.s_hi = t.empty((self.buf_cap, REC), dtype=t.float64, device=self.device)

    def local_maxd(self):
        return self.bdm.bdm_slab_local_maxd(self.h)

    def max_disp(self):
        return float(self.params.max_disp)

    def box_edge_min(self):
        return float(self.params.box_edge_min)

    def set_box_edge(self, L):
        self.bdm.bdm_slab_set_box_edge(self.h, L)

    def local_extents(self):
        return self.bdm.bdm_slab_local_extents(self.h)

    def pack(self, what, xb, xe):
        while True:
            rc, nlo, nhi = self.bdm.bdm_slab_pack(self.h, what, xb, xe, self.s_lo, self.s_hi, self.buf_cap)
            if rc == self.bdm.BDM_OK:
                return self.s_lo[:nlo], self.s_hi[:nhi]
            self.buf_cap = int(max(nlo, nhi) * 1.25) + 1024
            self._alloc()

    def split(self, xb, xe):
        if not hasattr(self, "info"):
            self.info = self.torch.zeros(12, dtype=self.torch.int64, device=self.device)
        self.bdm.bdm_slab_split(self.h, xb, xe, self.s_lo, self.s_hi, self.buf_cap, self.info)
        return self.s_lo, self.s_hi, self.info

    def commit(self, n_stay):
        self.bdm.bdm_slab_commit(self.h, n_stay)

    def grow_buffers(self, need):
        self.buf_cap = int(need * 1.25) + 1024
        self._alloc()

    def step(self, glo, ghi, xb, xe, recv_lo, recv_hi, want_dp=False):
        self.bdm.bdm_slab_step(self.h, glo, ghi, xb, xe, recv_lo, recv_lo.shape[0], recv_hi, recv_hi.shape[0],
                               want_dp)

    def add(self, recv_lo, recv_hi):
        self.bdm.bdm_slab_add(self.h, recv_lo, recv_lo.shape[0], recv_hi, recv_hi.shape[0])

    def owned(self):
        ids, pos = self.bdm.bdm_slab_get(self.h, self.bdm.BDM_OWNED_POSITIONS)
        return ids.cpu().numpy(), pos.cpu().numpy()

    def last_dp(self):
        ids, dp = self.bdm.bdm_slab_get(self.h, self.bdm.BDM_LAST_DISPLACEMENTS)
        return ids.cpu().numpy(), dp.cpu().numpy()


# --------------------------------------------------------------------------------- the protocol
HALO, MIGRANTS = 0, 1


class SlabDriver:
    """Runs the per-step protocol over the local slabs `engines` (engine k is slab comm.slab_ids()[k])."""

    def __init__(self, engines, comm, bounds, fused: bool | None = None):
        self.engines = engines
        self.comm = comm
        self.bounds = bounds
        self.slabs = [(bounds[g], bounds[g + 1]) for g in comm.slab_ids()]
        # single-sync protocol: needs every inner slab at least 2 boxes wide (so that an emigrant
        # never lands in a layer that is a third rank's ghost layer) and engines that can split
        inner = [b - a for a, b in zip(bounds[1:-2], bounds[2:-1])]
        L = comm.allreduce_max([e.local_maxd() for e in engines])  # O1 over all ranks
        L = max([L] + [e.box_edge_min() for e in engines if hasattr(e, "box_edge_min")])
        for e in engines:
            e.set_box_edge(L)
        self.L = L
        # the single-sync protocol also needs every step to move an agent by less than one box
        # (|dp| <= max_disp (1 + 4u) < L): only then are emigrants and next ghosts confined to the
        # two boundary layers k_slab_split scans
        small_moves = all(e.max_disp() < L * (1.0 - 2.0 ** -20) for e in engines if hasattr(e, "max_disp"))
        ok = all(w >= 2 for w in inner) and all(hasattr(e, "split") for e in engines) and small_moves
        self.fused = ok if fused is None else (fused and ok)
        self.next_ghosts = None
        self.migrated = 0  # agents moved between slabs by step() (diagnostics)
        self.settle()

    def migrate(self, count_global: bool = False):
        """Send emigrants to g-1 / g+1 and append the immigrants.  Returns the number of agents moved
        (globally when count_global -- an extra allreduce only the setup needs)."""
        sends = [e.pack(MIGRANTS, xb, xe) for e, (xb, xe) in zip(self.engines, self.slabs)]
        local = sum(s[0].shape[0] + s[1].shape[0] for s in sends)
        moved = self.comm.allreduce_sum([np.array([local], np.int64)])[0] if count_global else local
        recvs = self.comm.exchange(sends)
        for e, (rl, rh) in zip(self.engines, recvs):
            e.add(rl, rh)
        return int(moved)

    def settle(self, max_rounds: int | None = None):
        """Move every agent to its owner (agents hop one slab per round)."""
        rounds = 0
        while self.migrate(count_global=True) > 0:
            rounds += 1
            if rounds > (max_rounds or len(self.bounds)):
                raise RuntimeError("agents did not settle in their slabs")
        self.next_ghosts = None  # the next fused step primes its ghosts and extents
        return rounds

    def prime(self):
        """Extents and ghosts for the next step of the single-sync protocol (legacy exchanges)."""
        exts = [e.local_extents() for e in self.engines]
        self.glo, self.ghi = self.comm.allreduce_extents(exts)
        halos = [e.pack(HALO, xb, xe) for e, (xb, xe) in zip(self.engines, self.slabs)]
        self.next_ghosts = [(gl.clone(), gh.clone()) for gl, gh in self.comm.exchange(halos)]

    def step(self, want_dp: bool = False):
        """One protocol step.  Single-sync protocol: the exchange of the previous step's results (split,
        counts + extents, payloads, commit, immigrants, next ghosts) runs first, then the slab step;
        after it every agent is still owned by the rank that stepped it (an emigrant moves at the next
        exchange), so the owned sets partition the population between steps."""
        if not self.fused:
            return self.step_legacy(want_dp)
        if self.next_ghosts is None:
            self.prime()
        else:
            self.exchange()
        self.ghosts = sum(gl.shape[0] + gh.shape[0] for gl, gh in self.next_ghosts)
        for e, (xb, xe), (gl, gh) in zip(self.engines, self.slabs, self.next_ghosts):
            e.step(self.glo, self.ghi, xb, xe, gl, gh, want_dp)
        self.stepped = True

    def exchange(self):
        """Steps 2-4 of the single-sync protocol after a slab step (one host round trip)."""
        while True:
            splits = [e.split(xb, xe) for e, (xb, xe) in zip(self.engines, self.slabs)]
            outs = self.comm.exchange_split(splits)
            if not outs[0]["any_overflow"]:
                break
            for e, o in zip(self.engines, outs):  # some rank's buffers were too small: cancel, grow, redo
                e.commit(-1)
                e.grow_buffers(max(o["mig_lo"] + o["halo_lo"], o["mig_hi"] + o["halo_hi"]))
        ghosts = []
        for e, (s_lo, s_hi, _), o in zip(self.engines, splits, outs):
            # this rank's emigrants stay on as ghosts of the next step (they sit in the neighbour's
            # boundary layer); copied before the buffers are reused
            gl = self._cat(o["halo_in_lo"], s_lo[: o["mig_lo"]])
            gh = self._cat(o["halo_in_hi"], s_hi[: o["mig_hi"]])
            e.commit(o["n_stay"])
            e.add(o["imm_lo"], o["imm_hi"])
            self.migrated += o["mig_lo"] + o["mig_hi"]
            ghosts.append((gl, gh))
        self.next_ghosts = ghosts
        self.glo, self.ghi = outs[0]["glo"], outs[0]["ghi"]

    @staticmethod
    def _cat(a, b):
        import torch

        return torch.cat([a, b]) if b.shape[0] else a.clone()

    def step_legacy(self, want_dp: bool = False):
        exts = [e.local_extents() for e in self.engines]
        glo, ghi = self.comm.allreduce_extents(exts)
        halos = [e.pack(HALO, xb, xe) for e, (xb, xe) in zip(self.engines, self.slabs)]
        ghosts = self.comm.exchange(halos)
        self.ghosts = sum(gl.shape[0] + gh.shape[0] for gl, gh in ghosts)
        for e, (xb, xe), (gl, gh) in zip(self.engines, self.slabs, ghosts):
            e.step(glo, ghi, xb, xe, gl, gh, want_dp)
        self.migrated += self.migrate()


def layer_work(pos: np.ndarray, inv: float, x0: int, nx: int) -> np.ndarray:
    """Estimated work per box-x layer (cut by work, not by count).  An agent costs a
    fixed part (sort, displacement) plus a part proportional to its 27-box candidates, which scale
    with the occupancy n_b of its box: cost_i ~ 1 + c_i / c_mean with c_i ~ n_b(i).  Per layer:
    sum_b n_b + sum_b n_b^2 / (sum_all n_b^2 / N)."""
    b = np.floor(pos * inv).astype(np.int64)
    b -= b.min(axis=0)
    dims = b.max(axis=0) + 1
    key = (b[:, 0] * dims[1] + b[:, 1]) * dims[2] + b[:, 2]
    uk, cnt = np.unique(key, return_counts=True)
    layer = (uk // (dims[1] * dims[2])).astype(np.int64)
    cnt = cnt.astype(np.float64)
    n = np.bincount(layer, weights=cnt, minlength=nx)[:nx]
    sq = np.bincount(layer, weights=cnt * cnt, minlength=nx)[:nx]
    mean_sq = sq.sum() / max(len(pos), 1)
    return n + (sq / mean_sq if mean_sq > 0 else 0.0)


def initial_bounds(pos: np.ndarray, diam: np.ndarray, world: int, box_edge_min: float = 0.0,
                   weighted: bool = True):
    """Setup helper (outside the hot path): global L and work-balanced (weighted, default) or
    count-balanced bounds from the full population known to every rank (the bench generates the
    whole seeded population on every rank)."""
    L = max(float(diam.max()), box_edge_min)  # the engines' box edge (set_box_edge applies box_edge_min too)
    inv = 1.0 / (L * (1.0 + 2.0 ** -30))
    bx = np.floor(pos[:, 0] * inv).astype(np.int64)
    x0 = int(bx.min())
    hist = np.bincount(bx - x0)
    w = layer_work(pos, inv, x0, len(hist)) if weighted and world > 1 and len(pos) else None
    return choose_bounds(hist, x0, world, w), bx
