#!/usr/bin/env python
"""Steady-state steps of one config between cudaProfilerStart/Stop, for
`ncu --profile-from-start off` launch lists and kernel captures (warm-up excluded).

  python tools/profile_step.py [--config 3] [--steps 2] [--warmup 3]
"""
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
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--warmup", type=int, default=3)
a = ap.parse_args()
pos, diam = bdm_inputs.make_config(a.config)
h = bdm.bdm_init(torch.from_numpy(pos).cuda(), torch.from_numpy(diam).cuda(), stream=torch.cuda.current_stream())
bdm.bdm_mech_step(h, a.warmup)
bdm.bdm_sync(h)
torch.cuda.synchronize()
torch.cuda.profiler.start()
bdm.bdm_mech_step(h, a.steps)
bdm.bdm_sync(h)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled", a.steps, "steps of cfg", a.config, "n =", len(diam))
