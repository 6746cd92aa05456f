"""cfg4 (2e8 agents, device-generated): slow-path agents per step and the bench-style pass times."""
import sys
sys.path.insert(0, ".")
import torch
import bdm_inputs
import paper_2006_06775_b200 as bdm

bdm.load_library()
n = bdm_inputs.CFG_N[4]
lo, hi = bdm_inputs.box_of(4, n)
pos = torch.empty((n, 3), dtype=torch.float64, device="cuda")
diam = torch.empty(n, dtype=torch.float64, device="cuda")
bdm.bdm_generate_uniform(4, 0, n, lo, hi, 8.0, 12.0, pos, diam)
torch.cuda.synchronize()
h = bdm.bdm_init(pos, diam, bdm.bdm_params_default())
del pos, diam
for s in range(4):
    bdm.bdm_mech_step(h, 1)
    bdm.bdm_sync(h)
    print("step", s, bdm.bdm_get_path_stats(h), flush=True)
