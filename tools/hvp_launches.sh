#!/bin/bash
# per-kernel launch times of HVP batches on case9241 (ncu, serialized)
OUT=gpurun_out/${1:-hl}; mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python tools/prof_hvp.py case9241pegase 1024 2 > $OUT/log 2>&1
python tools/launch_summary.py $OUT/launches.csv > $OUT/summary.txt; cat $OUT/summary.txt
