#!/bin/bash
# A/B of k_blk knobs on case9241 (step probe, mask only)
OUT=gpurun_out/${1:-ab}; mkdir -p $OUT
for v in "base:" "nopf:RH_DEBUG=4096" "g4:RH_KBLK_GROUP=4" "g4nopf:RH_KBLK_GROUP=4 RH_DEBUG=4096" "g1:RH_KBLK_GROUP=1"; do
  tag=${v%%:*}; envs=${v#*:}
  env PROBE_TAG=$tag $envs timeout 300 python tools/step_probe.py --mask-only case9241pegase >> $OUT/ab.txt 2>&1
done
cat $OUT/ab.txt
