#!/bin/bash
# All BASELINE configs on 1 B200 (bench.py per case, oracle baseline included for the small ones)
TAG=${1:-sweep}; OUT=gpurun_out/$TAG; mkdir -p $OUT
for c in case9 case118 case1354pegase case2869pegase case9241pegase; do
  timeout 900 python bench.py --case $c --cpu-cols 512 > $OUT/sweep_$c.json 2> $OUT/sweep_$c.err
done
ls -la $OUT
