"""Soak check: many steps in one call (deferred builds, synchronised every 8) and in single-step calls,
bit-compared with the oracle's trajectory (cfg2, 10^6 agents, dt 1 and 0.1)."""
import sys
import time
sys.path.insert(0, ".")
import numpy as np
import bdm_inputs
import oracle
import paper_2006_06775_b200 as bdm

bdm.load_library()
pos, diam = bdm_inputs.make_config(2)
for dt, steps in ((1.0, 200), (0.1, 100)):
    t0 = time.time()
    po, _ = oracle.run(pos, diam, steps, oracle.params(dt=dt))
    t1 = time.time()
    h = bdm.bdm_init(pos, diam, bdm.bdm_params_default(dt=dt))
    bdm.bdm_mech_step(h, steps)
    p = bdm.bdm_get_positions(h)
    same = np.array_equal(p, po)
    h2 = bdm.bdm_init(pos, diam, bdm.bdm_params_default(dt=dt))
    for _ in range(steps // 10):
        bdm.bdm_mech_step(h2, 10)
    same2 = np.array_equal(bdm.bdm_get_positions(h2), po)
    print(f"dt={dt} steps={steps}: one call equal={same}, 10-step calls equal={same2}, "
          f"max|diff|={np.abs(p - po).max():.3e}, oracle {t1 - t0:.0f} s", flush=True)
