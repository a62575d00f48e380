#!/bin/bash
OUT=gpurun_out/${1:-pk}; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_blk -s 2 -c 4 \
   -o $OUT/kblk python tools/prof_hvp.py case9241pegase 1024 1 > $OUT/ncu.log 2>&1
python tools/ncu_summary.py $OUT/kblk.ncu-rep > $OUT/ncu_summary.txt 2>&1
cat $OUT/ncu_summary.txt
