#!/bin/sh
# A/B the cfg5 solver microbenchmark across library builds, interleaved:
#   tools/ab_cfg5.sh <lib.so|default|nopack> ... (run on the GPU box)
# "nopack" = the default library with OCTF_NO_PACK=1 (slot sample positions),
# "nomorton" = with OCTF_NO_MORTON=1 (frozen leaf-block list by base slot)
for rep in 1 2; do
  for lib in "$@"; do
    unset OCTF_NO_PACK OCTF_NO_MORTON
    case "$lib" in
      default) unset OCTF_LIB_PATH ;;
      nopack) unset OCTF_LIB_PATH; export OCTF_NO_PACK=1 ;;
      nomorton) unset OCTF_LIB_PATH; export OCTF_NO_MORTON=1 ;;
      *) export OCTF_LIB_PATH=$PWD/$lib ;;
    esac
    printf '%s ' "$lib"
    timeout 900 python tools/cfg5_bench.py ${CFG5_ARGS} 2>/dev/null | python -c "
import json, sys
D = json.load(sys.stdin)
print(' '.join('%s %.3f/%.3f %.3f' % (k, D[k]['kernel_ms'], D[k]['ms_per_step'], D[k]['frac_of_measured_hbm']) for k in ('descent_fp32', 'pd_fp32') if k in D))"
  done
done
