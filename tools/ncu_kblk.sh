#!/bin/bash
# ncu --set full of the k_blk launches of one Cartesian batch (current build)
OUT=gpurun_out/${1:-ncukblk}; shift; mkdir -p $OUT
env "$@" timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_blk \
   -o $OUT/kblk python tools/prof_hvp.py case9241pegase 1024 3 cartesian > $OUT/ncu.log 2>&1
tail -3 $OUT/ncu.log
