#!/bin/sh
# ncu --set full captures of the cfg5 descent and primal-dual leaf kernels
# (one launch each, after two warm passes):  sh tools/ncu_full_cfg5.sh <out>
O=${1:-gpurun_out/ncu}
mkdir -p $O
timeout 600 python tools/profile_cfg5.py --passes 3 > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:k_leaf_pass -s 2 -c 1 -o $O/ncu_leaf_cfg5 \
  python tools/profile_cfg5.py --only descent --passes 3 > $O/ncu_leaf.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:k_pd_pass -s 2 -c 1 -o $O/ncu_pd_cfg5 \
  python tools/profile_cfg5.py --only pd --passes 3 > $O/ncu_pd.log 2>&1
