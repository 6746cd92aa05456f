#!/usr/bin/env python
"""NEXT-3 measurement: soma clustering workload on one GPU.

Workload ("soma"): N agents uniform in a cube at 1e-3 um^-3 (counter hash, seed 7), D ~ U[8,12),
types 50/50 (counter hash), two substances on a lattice of spacing 12 um covering the cube plus two
nodes of padding, D_diff = 20 um^2/step, decay 0.01/step, dt = 1, secretion 1/agent/step, chemotaxis
0.5 um/step.  Times K steps with fields (secretion + diffusion + chemotaxis + mechanics) and, on
the same positions, K mechanics-only steps; the difference is the cost of the field operations.

  python tools/soma_bench.py [--n 2000000] [--steps 10] [--warmup 3]
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
ap.add_argument("--n", type=int, default=2_000_000)
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--warmup", type=int, default=3)
a = ap.parse_args()
side = (a.n / 1e-3) ** (1.0 / 3.0)
ids = np.arange(a.n)
pos, diam = bdm_inputs.uniform_population(7, ids, (0.0, 0.0, 0.0), (side, side, side), 8.0, 12.0)
types = (bdm_inputs.uniform01(7, ids, 5) < 0.5).astype(np.int8)
hsp = 12.0
dims = (int(side / hsp) + 5,) * 3
origin = (-2 * hsp,) * 3
stream = torch.cuda.current_stream()


def timed(with_fields):
    h = bdm.bdm_init(torch.from_numpy(pos).cuda(), torch.from_numpy(diam).cuda(), stream=stream)
    if with_fields:
        bdm.bdm_set_fields(h, hsp, origin, dims, 20.0, 0.01, 1.0, 1.0, 0.5, torch.from_numpy(types).cuda())
    bdm.bdm_mech_step(h, a.warmup)
    bdm.bdm_sync(h)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    bdm.bdm_mech_step(h, a.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    h.close()
    return ms


ms_f = timed(True)
ms_m = timed(False)
nn = dims[0] * dims[1] * dims[2]
bytes_fields = 2 * nn * 20  # per field: read c 8 + count 4, write 8 (secretion fused into the stencil)
print(json.dumps({"workload": f"soma: {a.n} agents at 1e-3/um^3, 2 substances on {dims} nodes (h={hsp} um)",
                  "value": a.n / (ms_f / 1e3), "unit": "agent-updates/s", "ms_per_step": ms_f,
                  "mechanics_only_ms_per_step": ms_m, "fields_ms_per_step": ms_f - ms_m,
                  "lattice_nodes": nn, "diffusion_algorithmic_bytes_per_step": bytes_fields}))
