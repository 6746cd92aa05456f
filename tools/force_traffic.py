#!/usr/bin/env python
"""Write profiles/r02_force_traffic.json (DRAM bytes of the force-phase kernels per step, read by
bench.py as roofline.traffic) from an ncu --set full capture of k_half_search + k_half_sum, or, with
--rebuild, profiles/r02_rebuild_traffic.json from the capture of the rebuild kernels (bench.py's
step_hbm: the whole step's measured DRAM bytes against HBM).

  python tools/force_traffic.py gpurun_out/r02_half.ncu-rep
  python tools/force_traffic.py --rebuild gpurun_out/r02_rebuild.ncu-rep"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
TSCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1, "msecond": 1}

rebuild = sys.argv[1] == "--rebuild"
rep = sys.argv[-1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
ks = []
for row in r[2:]:
    d, u = dict(zip(r[0], row)), dict(zip(r[0], r[1]))
    num = lambda k, sc: float(d[k].replace(",", "")) * sc[u[k]]  # noqa: E731
    ks.append({"kernel": d["Kernel Name"].split("(")[0].replace("bdm::", ""),
               "dram_bytes_read": int(num("dram__bytes_read.sum", SCALE)),
               "dram_bytes_write": int(num("dram__bytes_write.sum", SCALE)),
               "duration_ms_under_ncu": num("gpu__time_duration.sum", TSCALE)})
if rebuild:
    out = {"kernels": ks, "workload": "cfg3, steady-state build (tools/profile_step.py --steps 2)",
           "source": f"ncu --set full --clock-control none ({rep}); summary profiles/r02_rebuild_kernels_cfg3.txt",
           "kernel": "rebuild: table zero, key pass, scans, scatter, place", "n_agents": 20_000_000,
           "dram_bytes_read": sum(k["dram_bytes_read"] for k in ks),
           "dram_bytes_write": sum(k["dram_bytes_write"] for k in ks)}
    with open(os.path.join(ROOT, "profiles", "r02_rebuild_traffic.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))
    sys.exit(0)
out = {"kernels": ks,
       "workload": "cfg3, steady-state step (tools/profile_step.py --steps 2, first step captured: no dp write, "
                   "as in bench.py's timed mech_step(K))",
       "source": f"ncu --set full --clock-control none ({rep}); summary profiles/r02_half_kernels_cfg3.txt",
       "kernel": "force phase: k_half_search + k_half_sum",
       "n_agents": 20_000_000,
       "dram_bytes_read": sum(k["dram_bytes_read"] for k in ks),
       "dram_bytes_write": sum(k["dram_bytes_write"] for k in ks)}
with open(os.path.join(ROOT, "profiles", "r02_force_traffic.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out, indent=1))
