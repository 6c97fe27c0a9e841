#!/bin/sh
# Build tuning variants of the library next to the default one:
#   tools/build_variants.sh LEAF_MINB 2 3 4 5   (or PD_MINB 1 2 3 4)
set -e
cd "$(dirname "$0")/../paper_1608_07411_b200/csrc"
knob=${1:-LEAF_MINB}
shift || true
for mb in ${@:-2 3 4 5}; do
  make -s -j8 $knob=$mb OUT=../../build/liboctfuse_${knob}$mb.so \
       OBJDIR=../../build/obj_${knob}$mb
done
