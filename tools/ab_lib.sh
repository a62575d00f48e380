#!/bin/bash
# A/B of two library builds (step probe): current build vs exp_libs/<name>.so
OUT=${1:-ablib}; shift
cp paper_2201_00241_b200/libredhess.so /tmp/cur_lib.so
for name in "$@"; do
  bash tools/ab_step.sh $OUT "cur:X=1"
  cp exp_libs/$name.so paper_2201_00241_b200/libredhess.so
  bash tools/ab_step.sh $OUT "$name:X=1"
  cp /tmp/cur_lib.so paper_2201_00241_b200/libredhess.so
done
