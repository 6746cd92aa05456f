"""Multi-GPU front end of bench.py: one process per GPU, each owning one rank of libbdm's
distributed runtime (bdm_init_dist).  Argument marshalling and process plumbing
only: the partition, halo exchange and migration run inside libbdm.so (NCCL + CUDA kernels).

north_star: "Across the 8 GPUs of one box the domain is split into x-slabs.  Each step does a halo
exchange of boundary-box agents and migrates agents that cross slab boundaries, using NCCL
send/recv over NVLink."  torch.distributed carries only the communicator id, barriers and the
max-over-ranks timing.
"""
from __future__ import annotations

import os
import socket
import subprocess
import sys

import numpy as np


def torchrun_cmd(script: str, argv: list[str], nproc: int, port: int | None = None) -> list[str]:
    """The command that re-launches `script argv` as `nproc` ranks on this node (127.0.0.1)."""
    if port is None:
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
            "--master-addr=127.0.0.1", f"--master-port={port}", script] + list(argv)


def relaunch(script: str, argv: list[str], nproc: int) -> int:
    """bench.py --gpus N started without torchrun: run it under torchrun with N ranks (NCCL init
    logging on, so the rank count is visible) and pass its output through."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return subprocess.call(torchrun_cmd(script, argv, nproc), env=env)


def id_share(n: int, rank: int, world: int) -> tuple[int, int]:
    """The contiguous id range [a, b) a rank generates (an arbitrary initial distribution: the
    library redistributes every agent to the owner of its slab at init)."""
    return n * rank // world, n * (rank + 1) // world


def broadcast_uid(dist, bdm, device):
    """Rank 0's 128-byte NCCL communicator id, broadcast over torch.distributed."""
    import torch

    rank = dist.get_rank()
    raw = bdm.bdm_nccl_unique_id() if rank == 0 else bytes(128)
    t = torch.tensor(list(raw), dtype=torch.uint8, device=device)
    dist.broadcast(t, 0)
    return bytes(t.cpu().tolist())


def rank_inputs(bdm, torch, bdm_inputs, cfg: int, n: int, rank: int, world: int, dev, stream):
    """This rank's share of a config as device tensors (ids int64, pos, diam).  Counter-hash configs
    (1, 4, 5) are generated on the device for the rank's id range only (K0); cfg2 / cfg3 come from
    the host generator (the whole seeded population, then the rank's id range)."""
    a, b = id_share(n, rank, world)
    m = b - a
    ids = torch.arange(a, b, dtype=torch.int64, device=dev)
    if cfg in (1, 4, 5):
        lo, hi = bdm_inputs.box_of(cfg, n) if cfg != 1 else bdm_inputs.box_of(1)
        pos = torch.empty((m, 3), dtype=torch.float64, device=dev)
        diam = torch.empty(m, dtype=torch.float64, device=dev)
        bdm.bdm_generate_uniform(cfg, a, m, lo, hi, 8.0, 12.0, pos, diam, stream)
        torch.cuda.synchronize(dev)
        return ids, pos, diam
    pos_h, diam_h = bdm_inputs.make_config(cfg, n if n != bdm_inputs.CFG_N[cfg] else None)
    return (ids, torch.from_numpy(np.ascontiguousarray(pos_h[a:b])).to(dev),
            torch.from_numpy(np.ascontiguousarray(diam_h[a:b])).to(dev))
