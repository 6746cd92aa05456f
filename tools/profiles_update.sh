# regenerate the profiles/ summaries from the gpurun_out/ captures of tools/gpu/profile_round.sh (run here)
set -e
cd "$(dirname "$0")/.."
python tools/ncu_summary.py launches gpurun_out/bench_launches.csv > profiles/r01_launches_steady_cfg3.txt
cp gpurun_out/bench_launches.csv profiles/r01_bench_launches_cfg3.csv
python tools/ncu_summary.py kernel gpurun_out/half.ncu-rep > profiles/r01_half_kernels_cfg3.txt
python tools/ncu_summary.py kernel gpurun_out/rebuild.ncu-rep > profiles/r01_rebuild_kernels_cfg3.txt
python tools/force_traffic.py gpurun_out/half.ncu-rep > /dev/null
python tools/ncu_summary.py launches gpurun_out/nb_launches.csv > profiles/r01_neurite_launches.txt
python tools/ncu_summary.py kernel gpurun_out/elu.ncu-rep > profiles/r01_neurite_kernels.txt
echo profiles updated
