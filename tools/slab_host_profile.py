#!/usr/bin/env python
"""Host-side profile of the x-slab protocol at one rank (torchrun --nproc-per-node 1): GPU time of
one protocol step vs the wall time spent in each host phase (where the GPU may idle).

  python -m torch.distributed.run --nproc-per-node 1 --master-addr 127.0.0.1 tools/slab_host_profile.py"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bdm_inputs  # noqa: E402
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import slab_protocol as bdist  # noqa: E402

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
rank, world = dist.get_rank(), dist.get_world_size()
pos, diam = bdm_inputs.make_config(int(os.environ.get("CFG", "3")))
bounds, bx = bdist.initial_bounds(pos, diam, world)
mine = np.flatnonzero((bx >= bounds[rank]) & (bx < bounds[rank + 1]))
cap = int(len(mine) * 1.3) + 4096
stream = torch.cuda.current_stream()
eng = bdist.GpuSlabEngine(torch.from_numpy(mine).to(dev), torch.from_numpy(pos[mine]).to(dev),
                          torch.from_numpy(diam[mine]).to(dev), cap, stream=stream)
drv = bdist.SlabDriver([eng], bdist.TorchComm(dev), bounds)
for _ in range(3):
    drv.step()
torch.cuda.synchronize()
# wrap the phases
phases = {}
orig_ex = drv.comm.exchange_split


def timed(name, f):
    def g(*a, **k):
        t = time.perf_counter()
        r = f(*a, **k)
        phases[name] = phases.get(name, 0.0) + time.perf_counter() - t
        return r
    return g


drv.comm.exchange_split = timed("exchange_split (incl. the sync)", orig_ex)
eng.step = timed("engine.step (launches)", eng.step)
eng.split = timed("engine.split", eng.split)
eng.commit = timed("engine.commit", eng.commit)
eng.add = timed("engine.add", eng.add)
K = 20
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
K = int(os.environ.get("STEPS", K))
torch.cuda.profiler.start()
t0 = time.perf_counter()
e0.record(stream)
for _ in range(K):
    drv.step()
e1.record(stream)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
wall = time.perf_counter() - t0
print(f"fused={drv.fused} world={world} n_own={len(mine)}: {e0.elapsed_time(e1) / K:.3f} ms/step GPU, "
      f"{1e3 * wall / K:.3f} ms/step wall")
for k, v in phases.items():
    print(f"  {k:40s} {1e3 * v / K:8.3f} ms/step host")
dist.destroy_process_group()
