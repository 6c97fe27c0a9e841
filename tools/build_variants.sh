#!/bin/sh
# Build tuning variants of the library next to the default one.
set -e
cd "$(dirname "$0")/../paper_1608_07411_b200/csrc"
for mb in 2 3 4 5; do
  make -s -j8 LEAF_MINB=$mb OUT=../../build/liboctfuse_minb$mb.so \
       OBJDIR=../../build/obj_minb$mb
done
