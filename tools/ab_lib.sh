#!/bin/bash
# A/B of two builds of the library on the same box: swaps abtest/lib_old.so
# in for one run of the given command, then the current build.
#   bash tools/ab_lib.sh OUT "python tools/sweep_kernels.py"
OUT=$1; shift
LIB=paper_1407_6486_b200/lib/libpintlab_b200.so
cp $LIB /tmp/lib_new.so
for v in old new; do
  if [ $v = old ]; then cp abtest/lib_old.so $LIB; else cp /tmp/lib_new.so $LIB; fi
  echo "== $v" >> $OUT
  eval "$@" >> $OUT 2>&1
done
cp /tmp/lib_new.so $LIB
