#!/usr/bin/env python
"""NEXT-4 measurement: spheres + neurite elements on one GPU.

Workload: N spheres uniform at 1e-3 um^-3 (counter hash, seed 8), D ~ U[8,12); trees of 7 elements
(binary, 3 levels) rooted at random points, segments 5 um, diameters 2 um, resting length 5 um,
k_spring 10; K timed steps.  Reports updates/s counting spheres and distal points, and the time
with and without the elements (same spheres).

  python tools/neurite_bench.py [--n 2000000] [--trees 100000] [--steps 10]
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
ap.add_argument("--trees", type=int, default=100_000)
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--warmup", type=int, default=3)
a = ap.parse_args()
side = (a.n / 1e-3) ** (1.0 / 3.0)
pos, diam = bdm_inputs.uniform_population(8, np.arange(a.n), (0.0, 0.0, 0.0), (side,) * 3, 8.0, 12.0)
rng = np.random.default_rng(8)
T = a.trees
roots = rng.uniform(0.0, side, (T, 3))
dirs = rng.normal(size=(T, 7, 3))
dirs /= np.linalg.norm(dirs, axis=2)[:, :, None]
Q = np.zeros((T, 7, 3))
parent = [-1, 0, 0, 1, 1, 2, 2]
for j in range(7):
    P = roots if parent[j] < 0 else Q[:, parent[j]]
    Q[:, j] = P + 5.0 * dirs[:, j]
base = (np.arange(T) * 7)[:, None]
mother = np.where(np.array(parent)[None, :] < 0, -1, base + np.array(parent)[None, :]).reshape(-1)
dau = np.full((T, 7, 2), -1)
dau[:, 0] = base + np.array([1, 2])
dau[:, 1] = base + np.array([3, 4])
dau[:, 2] = base + np.array([5, 6])
E = 7 * T
stream = torch.cuda.current_stream()


def timed(with_neurites):
    h = bdm.bdm_init(torch.from_numpy(pos).cuda(), torch.from_numpy(diam).cuda(), stream=stream)
    if with_neurites:
        bdm.bdm_set_neurites(h, Q.reshape(-1, 3), np.full(E, 2.0), np.full(E, 5.0), np.repeat(roots, 7, axis=0),
                             mother, dau.reshape(-1, 2), 10.0)
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


ms_n = timed(True)
ms_s = timed(False)
print(json.dumps({"workload": f"{a.n} spheres at 1e-3/um^3 + {E} neurite elements ({T} 7-element trees)",
                  "value": (a.n + E) / (ms_n / 1e3), "unit": "updates/s (spheres + distal points)",
                  "ms_per_step": ms_n, "spheres_only_ms_per_step": ms_s}))
