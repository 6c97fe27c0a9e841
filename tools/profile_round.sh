#!/bin/sh
# One GPU-box profiling sweep (run under gpurun from the repo root):
# bench line, cfg5 microbenchmark, ncu launch list of the bench command, and
# ncu --set full captures of the descent and primal-dual leaf kernels.
# Each ncu pass runs only after the same command exited 0 without ncu.
set -u
O=gpurun_out/prof
mkdir -p $O
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err || exit 1
timeout 900 python tools/cfg5_bench.py > $O/cfg5.json 2> $O/cfg5.err || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 \
  -k regex:"k_leaf_pass|k_propagate|k_sum_stage|k_pd_pass" \
  --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity-mode \
  --no-pd > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:k_leaf_pass -s 3 -c 1 -o $O/ncu_leaf \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity-mode \
  --no-pd > $O/ncu_leaf.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:k_pd_pass -s 3 -c 1 -o $O/ncu_pd_cfg2 \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity-mode \
  > $O/ncu_pd_cfg2.log 2>&1
timeout 600 python tools/cfg5_bench.py --leaves 10000000 --only pd --steps 2 \
  > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:k_pd_pass -s 2 -c 1 -o $O/ncu_pd_cfg5 \
  python tools/cfg5_bench.py --leaves 10000000 --only pd --steps 2 \
  > $O/ncu_pd.log 2>&1
echo done
