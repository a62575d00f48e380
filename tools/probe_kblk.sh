#!/bin/bash
OUT=gpurun_out/${1:-pk}; mkdir -p $OUT
RH_DEBUG=8 timeout 300 python tools/diag.py case9241pegase > $OUT/diag_dbg8.txt 2>&1
python tools/kblk_prof.py gpurun_out/kblk_prof.bin > $OUT/kblk_prof.txt 2>&1
cat $OUT/kblk_prof.txt
