"""Child process of tests/test_gpu_ring.py and tests/test_gpu_switches.py: steps a population through
libbdm under the environment switches its parent set (read when the library loads, e.g. BDM_RING) and
checks the trajectory against the oracle's."""
import json
import sys

import numpy as np

import bdm_inputs
import oracle
import paper_2006_06775_b200 as bdm


def main():
    cfg, steps = int(sys.argv[1]), int(sys.argv[2])
    one_call = len(sys.argv) > 3 and sys.argv[3] == "one"
    bdm.load_library()
    pos, diam = bdm_inputs.make_config(cfg)
    h = bdm.bdm_init(pos, diam, bdm.bdm_params_default())
    paths = []
    if one_call:  # all steps in one bdm_mech_step call (deferred builds between them)
        bdm.bdm_mech_step(h, steps)
        paths.append(bdm.bdm_get_path_stats(h)["half"])
    else:
        for _ in range(steps):
            bdm.bdm_mech_step(h, 1)
            paths.append(bdm.bdm_get_path_stats(h)["half"])
    p = bdm.bdm_get_positions(h)
    po, _ = oracle.run(pos, diam, steps)
    print(json.dumps({"paths": paths, "equal": bool(np.array_equal(p, po)), "n": int(len(diam))}))


if __name__ == "__main__":
    main()
