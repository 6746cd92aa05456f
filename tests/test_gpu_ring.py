"""The banded force phase over a ring of pair rows (populations whose rows do not fit
beside the state, e.g. 10^9 agents on one GPU) against the CPU oracle, bit for bit.  The ring is forced
at small sizes with BDM_RING (read when libbdm loads, hence a child process per case): ring sizes that
cut the population into several bands, a ring too small for the grid's two-layer span (the step falls
back to k_force), and multi-step calls with deferred builds (BASELINE.json north_star parity contract;
DESIGN.md §3.3)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(cfg, steps, ring_log, mode="each"):
    env = dict(os.environ, BDM_RING=str(ring_log), PYTHONPATH=ROOT)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "ring_child.py"), str(cfg), str(steps), mode],
                         env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("mode", ["each", "one"])
def test_ring_cfg1_bands(mode):
    """configs[0] (4096 agents, two box-x layers ~600 agents) in bands of 1024 agents (a 2^11-row ring:
    four bands per step), 6 steps, one call per step or all in one call (deferred builds)."""
    r = child(1, 6, 11, mode)
    assert all(p == 2 for p in r["paths"]), r
    assert r["equal"], r


def test_ring_cfg2():
    """configs[1] (10^6 agents), a 2^18-row ring, 3 steps: bit-identical to the oracle's trajectory."""
    r = child(2, 3, 18)
    assert all(p == 2 for p in r["paths"]), r
    assert r["equal"], r


def test_ring_too_small_falls_back():
    """A ring smaller than two layers of configs[1]: every step takes k_force, results unchanged."""
    r = child(2, 2, 8)
    assert all(p == 0 for p in r["paths"]), r
    assert r["equal"], r
