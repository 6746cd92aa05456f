timeout 900 python tools/relax_experiment.py --config 3 --steps 60 --every 30 2>&1 | tail -2
cat > /tmp/ps.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import torch, bdm_inputs, paper_2006_06775_b200 as bdm
pos, diam = bdm_inputs.make_config(3)
tp, td = torch.from_numpy(pos).cuda(), torch.from_numpy(diam).cuda()
prm = bdm.bdm_params_default(); prm.flags |= bdm.BDM_SKIP_STATIONARY
h = bdm.bdm_init(tp, td, prm, stream=torch.cuda.current_stream())
bdm.bdm_mech_step(h, 60); bdm.bdm_sync(h); torch.cuda.synchronize()
torch.cuda.profiler.start(); bdm.bdm_mech_step(h, 2); bdm.bdm_sync(h); torch.cuda.synchronize(); torch.cuda.profiler.stop()
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/skip_launches.csv python /tmp/ps.py > /dev/null 2>&1; echo ncu rc=$?
