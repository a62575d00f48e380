#!/bin/bash
# Quick GPU check: the GPU parity suite and the step probe.
OUT=gpurun_out/${1:-quick}; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
timeout 600 python tools/step_probe.py > $OUT/step_probe.txt 2>&1
tail -3 $OUT/pytest_gpu.txt; cat $OUT/step_probe.txt
