#!/bin/sh
# A/B the cfg2 bench line (leaf kernel + step) across library builds,
# interleaved: tools/ab_bench.sh <lib.so|default> ...  (GPU box)
for rep in 1 2; do
  for lib in "$@"; do
    if [ "$lib" = default ]; then unset OCTF_LIB_PATH; else export OCTF_LIB_PATH=$PWD/$lib; fi
    printf '%s ' "$lib"
    timeout 600 python bench.py --no-e2e --no-cpu --no-parity-mode ${BENCH_ARGS} 2>/dev/null | tail -1 | python -c "
import json, sys
D = json.loads(sys.stdin.read())
pd = D.get('pd_mode', {})
print('step %.4f ms  leaf %.4f ms  frac %.3f  pd %.4f ms frac %.3f' % (D['ms_per_step'], D['roofline']['kernel_ms'], D['roofline']['frac'], pd.get('ms_per_step', 0), pd.get('roofline', {}).get('frac', 0)))"
  done
done
