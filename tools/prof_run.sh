#!/bin/bash
# ncu captures of the HVP kernels + the refactorization (one GPU; never multi-rank)
TAG=${1:-prof}; CASE=${2:-case9241pegase}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_blk|k_sep|k_for|k_muladd' -s 8 -c 8 \
   -o $OUT/hvp python tools/prof_hvp.py $CASE > $OUT/ncu_hvp.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_fact|k_assemble|k_sep_inverse' -c 6 \
   -o $OUT/fact python tools/prof_hvp.py $CASE 64 1 > $OUT/ncu_fact.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
   python tools/prof_hvp.py $CASE > $OUT/ncu_launch.log 2>&1
ls -la $OUT
