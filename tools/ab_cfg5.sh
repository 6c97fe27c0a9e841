#!/bin/sh
# A/B the cfg5 solver microbenchmark across library builds, interleaved:
#   tools/ab_cfg5.sh <lib.so|default> ... (run on the GPU box)
for rep in 1 2; do
  for lib in "$@"; do
    if [ "$lib" = default ]; then unset OCTF_LIB_PATH; else export OCTF_LIB_PATH=$PWD/$lib; fi
    printf '%s ' "$lib"
    timeout 900 python tools/cfg5_bench.py ${CFG5_ARGS} 2>/dev/null | python -c "
import json, sys
D = json.load(sys.stdin)
print(' '.join('%s %.3f/%.3f %.3f' % (k, D[k]['kernel_ms'], D[k]['ms_per_step'], D[k]['frac_of_measured_hbm']) for k in ('descent_fp32', 'pd_fp32') if k in D))"
  done
done
