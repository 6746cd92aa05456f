# regenerate the profiles/ summaries of round 2 from the gpurun_out/ captures of tools/gpu/profile_r02.sh (run here)
set -e
cd "$(dirname "$0")/.."
python tools/ncu_summary.py launches gpurun_out/r02_bench_launches.csv > profiles/r02_launches_steady_cfg3.txt
cp gpurun_out/r02_bench_launches.csv profiles/r02_bench_launches_cfg3.csv
python tools/ncu_summary.py kernel gpurun_out/r02_half.ncu-rep > profiles/r02_half_kernels_cfg3.txt
python tools/ncu_summary.py kernel gpurun_out/r02_rebuild.ncu-rep > profiles/r02_rebuild_kernels_cfg3.txt
python tools/force_traffic.py gpurun_out/r02_half.ncu-rep > /dev/null
python tools/force_traffic.py --rebuild gpurun_out/r02_rebuild.ncu-rep > /dev/null
python tools/ncu_summary.py launches gpurun_out/r02_dist_launches.csv > profiles/r02_dist_launches_cfg3_1rank.txt
cp gpurun_out/r02_fp64_microbench.txt profiles/r02_fp64_microbench.txt
echo profiles updated
