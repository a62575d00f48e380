#!/bin/bash
OUT=gpurun_out/${1:-kp}; mkdir -p $OUT
for g in 2 4; do
  RH_KBLK_GROUP=$g RH_DEBUG=8 timeout 300 python tools/prof_hvp.py case9241pegase 1024 2 > /dev/null 2>&1
  echo "group $g" >> $OUT/kblk_prof.txt; python tools/kblk_prof.py gpurun_out/kblk_prof.bin >> $OUT/kblk_prof.txt 2>&1
  RH_KBLK_GROUP=$g RH_DEBUG=4104 timeout 300 python tools/prof_hvp.py case9241pegase 1024 2 > /dev/null 2>&1
  echo "group $g no prefetch" >> $OUT/kblk_prof.txt; python tools/kblk_prof.py gpurun_out/kblk_prof.bin >> $OUT/kblk_prof.txt 2>&1
done
cat $OUT/kblk_prof.txt
