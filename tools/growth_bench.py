#!/usr/bin/env python
"""NEXT-2 measurement: cell growth and division workload on one GPU.

Workload ("cgd"): N0 agents uniform in a cube at 1e-3 um^-3 (counter hash, seed 6),
D ~ U[8, 12), growth 0.25 um/step, division at D >= 12 um; K timed steps after W warm-up steps.
Reports agent-updates/s (sum over steps of the population mechanically updated / device time),
the population growth and the share of the growth + division kernels.

  python tools/growth_bench.py [--n 4000000] [--steps 10] [--warmup 3]
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
ap.add_argument("--n", type=int, default=4_000_000)
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--growth", type=float, default=0.25)
ap.add_argument("--div", type=float, default=12.0)
a = ap.parse_args()
side = (a.n / 1e-3) ** (1.0 / 3.0)
pos, diam = bdm_inputs.uniform_population(6, np.arange(a.n), (0.0, 0.0, 0.0), (side, side, side), 8.0, 12.0)
stream = torch.cuda.current_stream()
h = bdm.bdm_init(torch.from_numpy(pos).cuda(), torch.from_numpy(diam).cuda(), stream=stream)
bdm.bdm_set_growth(h, a.growth, a.div, 6)
bdm.bdm_reserve(h, 4 * a.n)
bdm.bdm_set_timing(h, True)
for _ in range(a.warmup):
    bdm.bdm_mech_step(h, 1)
bdm.bdm_sync(h)
bdm.bdm_get_timing(h)
n_start = bdm.bdm_get_count(h)[0]
updates = 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(stream)
for _ in range(a.steps):
    updates += bdm.bdm_get_count(h)[0]
    bdm.bdm_mech_step(h, 1)
e1.record(stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
tm = bdm.bdm_get_timing(h)
n_end = bdm.bdm_get_count(h)[0]
print(json.dumps({"workload": f"cgd: {a.n} agents at 1e-3/um^3, D~U[8,12), growth {a.growth} um/step, division at {a.div} um",
                  "value": updates / (ms / 1e3), "unit": "agent-updates/s", "steps": a.steps,
                  "ms_per_step": ms / a.steps, "population": [n_start, n_end],
                  "grid_ms_per_step": tm["grid_ms"] / tm["steps"], "force_ms_per_step": tm["force_ms"] / tm["steps"],
                  "search_ms_per_step": tm.get("search_ms", 0.0) / tm["steps"],
                  "note": "force_ms includes the growth + division kernels (they run after the force kernel)"}))
