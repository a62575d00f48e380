#!/bin/bash
# separator Gauss-Jordan inverse: per-panel phase probe (RH_DEBUG=16, tools/gj_prof.py)
OUT=gpurun_out/${1:-gj}; mkdir -p $OUT
RH_DEBUG=16 timeout 300 python tools/diag.py case9241pegase > $OUT/diag16.txt 2>&1
python tools/gj_prof.py gpurun_out/gj_prof.bin | tee $OUT/gj.txt
