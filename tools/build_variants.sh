#!/bin/sh
# Build tuning variants of the library next to the default one:
#   tools/build_variants.sh LEAF_MINB 2 3 4 5   (or PD_MINB 1 2 3 4)
#   tools/build_variants.sh DEFS -DOCTF_STAGES=1 -DOCTF_STAGES=3
# -> build/liboctfuse_<knob><value>.so (objects under build/obj/, which
# does not travel to the GPU box)
set -e
cd "$(dirname "$0")/../paper_1608_07411_b200/csrc"
knob=${1:-LEAF_MINB}
shift || true
for mb in ${@:-2 3 4 5}; do
  tag=$(echo "${knob}${mb}" | tr -c 'A-Za-z0-9_\n' '_')
  make -s -j8 "$knob=$mb" OUT=../../build/liboctfuse_$tag.so \
       OBJDIR=../../build/obj/$tag
done
