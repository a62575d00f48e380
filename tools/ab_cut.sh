#!/bin/bash
# A/B of the unit-sweep cut factor (RH_CUT) on case9241: step probe, mask only
OUT=gpurun_out/${1:-abcut}; shift; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
tail -2 $OUT/pytest_gpu.txt
for c in "$@"; do
  RH_CUT=$c PROBE_TAG=cut$c timeout 300 python tools/step_probe.py case9241pegase >> $OUT/ab.txt 2>&1
done
cat $OUT/ab.txt
