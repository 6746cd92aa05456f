"""The run-time A/B switches of libbdm (read when the library loads, hence a child process each) leave
results unchanged: every variant of the step is bit-identical to the oracle (
BASELINE.json north_star parity contract).  BDM_PDL=0: no programmatic dependent launch; BDM_TZERO=0:
the build zeroes its own histogram; BDM_FUSE=0: no fused column pass (the build's own column pass);
BDM_PBOX=0: the key pass reads the state instead of the packed boxes; BDM_DEFER=0: every build
synchronised."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("env", ["BDM_PDL=0", "BDM_TZERO=0", "BDM_FUSE=0", "BDM_PBOX=0", "BDM_DEFER=0"])
@pytest.mark.parametrize("mode", ["each", "one"])
def test_switch_keeps_results(env, mode):
    k, v = env.split("=")
    e = dict(os.environ, PYTHONPATH=ROOT)
    e[k] = v
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "ring_child.py"), "1", "5", mode], env=e,
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert all(p == 1 for p in r["paths"]), r
    assert r["equal"], r
