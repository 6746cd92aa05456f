#!/usr/bin/env python
"""NEXT-1 measurement helper: how many agents still move as a population relaxes, and the step time
with and without the stationary-region skip at the same relaxed state.

  python tools/relax_experiment.py --config 2 --steps 300 --every 25
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
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--steps", type=int, default=300)
ap.add_argument("--every", type=int, default=25)
ap.add_argument("--adherence", type=float, default=0.1)
a = ap.parse_args()
pos, diam = bdm_inputs.make_config(a.config)
tp, td = torch.from_numpy(pos).cuda(), torch.from_numpy(diam).cuda()


def handle(skip):
    prm = bdm.bdm_params_default(adherence=a.adherence)
    if skip:
        prm.flags |= bdm.BDM_SKIP_STATIONARY
    h = bdm.bdm_init(tp, td, prm, stream=torch.cuda.current_stream())
    bdm.bdm_set_timing(h, True)
    return h


hs, hn = handle(True), handle(False)
for s in range(0, a.steps, a.every):
    for h in (hs, hn):
        bdm.bdm_get_timing(h)
        bdm.bdm_mech_step(h, a.every)
        bdm.bdm_sync(h)
    ts, tn = bdm.bdm_get_timing(hs), bdm.bdm_get_timing(hn)
    st = bdm.bdm_get_skip_stats(hs)
    same = bool(torch.equal(bdm.bdm_get_positions(hs), bdm.bdm_get_positions(hn)))
    print(f"steps {s + a.every:4d}: moved {st['moved'] / st['n']:.3f} searched {st['searched'] / st['n']:.3f} "
          f"ms/step skip {(ts['grid_ms'] + ts['force_ms']) / ts['steps']:.3f} "
          f"(force {ts['force_ms'] / ts['steps']:.3f}) no-skip {(tn['grid_ms'] + tn['force_ms']) / tn['steps']:.3f} "
          f"(force {tn['force_ms'] / tn['steps']:.3f}) identical={same}; skip passes search "
          f"{ts['search_ms'] / ts['steps']:.3f} sum {ts['sum_ms'] / ts['steps']:.3f}, no-skip "
          f"{tn['search_ms'] / tn['steps']:.3f} / {tn['sum_ms'] / tn['steps']:.3f}", flush=True)
