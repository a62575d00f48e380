#!/bin/bash
OUT=gpurun_out/${1:-tl}; mkdir -p $OUT
RH_DEBUG=1024 timeout 300 python tools/step_timeline.py case9241pegase 1024 > $OUT/timeline.txt 2>&1
tail -60 $OUT/timeline.txt
