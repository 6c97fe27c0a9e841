#!/bin/sh
# One GPU-box profiling sweep (run under gpurun from the repo root):
# bench line (cfg5 headline), ncu launch list of the bench step, and ncu
# --set full captures of the descent and primal-dual leaf kernels on cfg5.
# Each ncu pass runs only after the same command exited 0 without ncu.
#   sh tools/profile_round.sh [out-dir]
set -u
O=${1:-gpurun_out/prof}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err || exit 1
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu \
  --no-parity --no-cfg2 > $O/bench_short.json 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 \
  -k regex:"^k_" --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity \
  --no-cfg2 > $O/ncu_launch.log 2>&1
timeout 600 python tools/profile_cfg5.py --passes 3 > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:k_leaf_pass -s 2 -c 1 -o $O/ncu_leaf_cfg5 \
  python tools/profile_cfg5.py --only descent --passes 3 \
  > $O/ncu_leaf.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:k_pd_pass -s 2 -c 1 -o $O/ncu_pd_cfg5 \
  python tools/profile_cfg5.py --only pd --passes 3 \
  > $O/ncu_pd.log 2>&1
echo done
