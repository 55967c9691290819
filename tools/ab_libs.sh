#!/bin/bash
# A/B of several builds of the library on one box: runs CMD once per
# abtest/lib_<name>.so (swapped in for the run), then restores the current build.
#   bash tools/ab_libs.sh "name1 name2" "python tools/sweep_kernels.py | grep jor_rb"
LIB=paper_1407_6486_b200/lib/libpintlab_b200.so
cp $LIB /tmp/lib_cur.so
for v in $1; do
  cp abtest/lib_$v.so $LIB
  echo "== $v"
  eval "$2" 2>&1
done
cp /tmp/lib_cur.so $LIB
