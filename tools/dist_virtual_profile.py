#!/usr/bin/env python
"""One timed step of G virtual ranks between cudaProfilerStart/Stop (ncu --profile-from-start off launch
lists of the distributed runtime).  python tools/dist_virtual_profile.py [--ranks 8] [--config 3]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bdm_inputs  # noqa: E402
import paper_2006_06775_b200 as bdm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--ranks", type=int, default=8)
a = ap.parse_args()
pos, diam = bdm_inputs.make_config(a.config)
n = len(diam)
G = a.ranks
counts = [n * (r + 1) // G - n * r // G for r in range(G)]
st = torch.cuda.Stream()
h = bdm.bdm_init_dist_local(G, counts, torch.arange(n, dtype=torch.int64, device="cuda"),
                            torch.from_numpy(pos).cuda(), torch.from_numpy(diam).cuda(), stream=st)
bdm.bdm_mech_step(h, 3)
bdm.bdm_sync(h)
torch.cuda.synchronize()
torch.cuda.profiler.start()
bdm.bdm_mech_step(h, 2)
bdm.bdm_sync(h)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled 2 steps of", G, "virtual ranks, n =", n)
