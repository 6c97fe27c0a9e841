#!/bin/sh
# A/B the restructuring configurations across library builds, interleaved:
#   tools/ab_restructure.sh <lib.so|default> ...   (run on the GPU box)
# prints per build: cfg3 / cfg4 depth 9 / cfg4 depth 10 pass ms (a Python call
# per pass, timers on) and the leaf kernel's median ms
python tools/cfg3_bench.py --passes 2 --save-scene /tmp/ab_cfg3.pkl > /dev/null 2>&1
python tools/cfg3_bench.py --config cfg4 --depth 9 --passes 2 --save-scene /tmp/ab_cfg4.pkl > /dev/null 2>&1
for rep in 1 2; do
  for lib in "$@"; do
    case "$lib" in
      default) unset OCTF_LIB_PATH ;;
      *) export OCTF_LIB_PATH=$PWD/$lib ;;
    esac
    printf '%s ' "$lib"
    for cfg in "--load-scene /tmp/ab_cfg3.pkl" "--config cfg4 --depth 9 --load-scene /tmp/ab_cfg4.pkl" "--config cfg4 --depth 10"; do
      python tools/cfg3_bench.py $cfg --passes 30 2>/dev/null | python -c "
import json, sys
d = json.load(sys.stdin)
lm = sorted(p['leaf_ms'] for p in d['passes'][5:])
print('%.3f/%.3f' % (d['median_pass_ms'], lm[len(lm) // 2]), end=' ')"
    done
    echo
  done
done
