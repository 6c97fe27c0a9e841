#!/bin/sh
# interleaved A/B: base lib, new lib with fusion, new lib without fusion
for rep in 1 2 3; do
  for v in base new nofuse; do
    unset OCTF_LIB_PATH OCTF_NO_FUSED_PARENT
    [ $v = base ] && export OCTF_LIB_PATH=$PWD/build/lib_base.so
    [ $v = nofuse ] && export OCTF_NO_FUSED_PARENT=1
    printf '%s ' "$v"
    timeout 600 python bench.py --no-e2e --no-cpu --no-parity-mode 2>/dev/null | tail -1 | python -c "
import json, sys
D = json.loads(sys.stdin.read())
pd = D.get('pd_mode', {})
print('step %.4f ms  leaf %.4f ms  frac %.3f  pd %.4f ms frac %.3f' % (D['ms_per_step'], D['roofline']['kernel_ms'], D['roofline']['frac'], pd.get('ms_per_step', 0), pd.get('roofline', {}).get('frac', 0)))"
  done
done
