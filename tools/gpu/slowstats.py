"""cfg3: how many agents take the half-shell slow path per step, and the step's kernel times."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import bdm_inputs
import paper_2006_06775_b200 as bdm

bdm.load_library()
pos, diam = bdm_inputs.make_config(3)
h = bdm.bdm_init(pos, diam, bdm.bdm_params_default())
for s in range(4):
    bdm.bdm_mech_step(h, 1)
    bdm.bdm_sync(h)
    print("step", s, bdm.bdm_get_path_stats(h))
