#!/usr/bin/env python
"""Fixed cost of the distributed runtime's protocol per step: G virtual ranks of one process on one GPU
(bdm_init_dist_local; their kernels run one after another) against the single handle on the same
population.  (G-rank time - single time) / G ~ the per-rank, per-step fixed cost of the protocol.

  python tools/dist_virtual_bench.py [--config 3] [--ranks 1 2 4 8] [--steps 16]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bdm_inputs  # noqa: E402
import paper_2006_06775_b200 as bdm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--ranks", type=int, nargs="+", default=[1, 2, 4, 8])
ap.add_argument("--steps", type=int, default=16)
a = ap.parse_args()
pos, diam = bdm_inputs.make_config(a.config)
n = len(diam)
tp, td = torch.from_numpy(pos).cuda(), torch.from_numpy(diam).cuda()
st = torch.cuda.Stream()  # (a capturable stream: the distributed runtime replays its steady steps as graphs)


def timed(h, steps):
    bdm.bdm_mech_step(h, steps)  # warm-up (one chunk)
    bdm.bdm_sync(h)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    bdm.bdm_mech_step(h, steps)
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


h = bdm.bdm_init(tp, td, stream=st)
out = {"config": a.config, "n": n, "single_ms": timed(h, a.steps)}
h.close()
ids = torch.arange(n, dtype=torch.int64, device="cuda")
for G in a.ranks:
    counts = [n * (r + 1) // G - n * r // G for r in range(G)]
    hd = bdm.bdm_init_dist_local(G, counts, ids, tp, td, stream=st)
    ms = timed(hd, a.steps)
    s = bdm.bdm_get_stats(hd)
    out[f"virtual_{G}_ms"] = ms
    out[f"virtual_{G}_fixed_us_per_rank"] = 1e3 * (ms - out["single_ms"]) / G
    out[f"virtual_{G}_syncs"] = s["host_syncs"]
    cuts = bdm.bdm_get_cuts(hd)
    hd.close()
    torch.cuda.empty_cache()
    if G > 1:  # the same slabs as independent single handles (no ghosts, no protocol): sum of their steps
        L = float(diam.max())
        bx = np.floor(pos[:, 0] * (1.0 / (L * (1.0 + 2.0 ** -30)))).astype(np.int64)
        tot = 0.0
        for g in range(G):
            m = np.flatnonzero((bx >= cuts[g]) & (bx < cuts[g + 1]))
            if len(m) == 0:
                continue
            hs = bdm.bdm_init(torch.from_numpy(pos[m].copy()).cuda(), torch.from_numpy(diam[m].copy()).cuda(),
                              stream=st)
            tot += timed(hs, a.steps)
            hs.close()
        out[f"singles_{G}_sum_ms"] = tot
        out[f"virtual_{G}_protocol_us_per_rank"] = 1e3 * (out[f"virtual_{G}_ms"] - tot) / G
print(json.dumps(out))
