"""CPU tests of the multi-GPU front end (paper_2006_06775_b200/dist.py, bench.py --gpus N): the
torchrun relaunch, the per-rank id shares and the NCCL communicator id broadcast over a world-2
gloo group (127.0.0.1).  The distributed runtime itself needs CUDA (tests/test_gpu_dist.py)."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_torchrun_command():
    from paper_2006_06775_b200 import dist as bdist

    cmd = bdist.torchrun_cmd("/x/bench.py", ["--gpus", "8", "--steps", "3"], 8, port=12345)
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in cmd and "--master-addr=127.0.0.1" in cmd and "--master-port=12345" in cmd
    assert cmd[-4:] == ["--gpus", "8", "--steps", "3"] and cmd[-5] == "/x/bench.py"


@pytest.mark.parametrize("n", [0, 1, 7, 4096, 1_000_003])
def test_id_shares_partition_the_population(n):
    from paper_2006_06775_b200 import dist as bdist

    for world in range(1, 9):
        seen = np.zeros(n, np.int64)
        prev = 0
        for r in range(world):
            a, b = bdist.id_share(n, r, world)
            assert a == prev and a <= b
            seen[a:b] += 1
            prev = b
        assert prev == n and np.all(seen == 1)


def _uid_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2006_06775_b200 as bdm
    from paper_2006_06775_b200 import dist as bdist

    uid = bdist.broadcast_uid(dist, bdm, "cpu")
    out[rank] = uid.hex()
    dist.destroy_process_group()


def test_uid_broadcast_gloo_world2():
    """Rank 0's bdm_nccl_unique_id reaches rank 1 unchanged (what bench.py's ranks do before
    bdm_init_dist)."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_uid_worker, args=(2, port, out), nprocs=2, join=True)
    assert len(out[0]) == 256 and out[0] == out[1]


def test_bench_relaunches_under_torchrun(monkeypatch):
    """bench.py --gpus N without WORLD_SIZE re-runs itself under torchrun with N ranks and NCCL init
    logging (the rank count visible to the driver)."""
    import bench
    from paper_2006_06775_b200 import dist as bdist

    calls = []

    def fake_call(cmd, env=None):
        calls.append((cmd, env))
        return 0

    monkeypatch.setattr(subprocess, "call", fake_call)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2", "--warmup", "3"])
    assert bench.main() == 0
    cmd, env = calls[0]
    assert "--nproc-per-node=4" in cmd and cmd[-6:] == ["--gpus", "4", "--steps", "2", "--warmup", "3"]
    assert env["NCCL_DEBUG"] == "INFO" and env.get("NCCL_DEBUG_SUBSYS") == "INIT"
