#!/bin/bash
# Quick GPU check: parity tests + per-stage timing on all configs + k_blk per-tile probe.  One GPU.
OUT=gpurun_out/${1:-quick}; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
timeout 600 python tools/diag.py > $OUT/diag.txt 2>&1
RH_DEBUG=8 timeout 300 python tools/diag.py case9241pegase > $OUT/diag_dbg8.txt 2>&1
python tools/kblk_prof.py gpurun_out/kblk_prof.bin > $OUT/kblk_prof.txt 2>&1
tail -3 $OUT/pytest_gpu.txt; cat $OUT/diag.txt $OUT/kblk_prof.txt
