#!/bin/bash
# per-tile k_blk (MODE_U) phase probe (RH_DEBUG=8) under env variants "tag:ENV=.."
OUT=gpurun_out/${1:-kblkab}; shift; mkdir -p $OUT
for v in "$@"; do
  tag=${v%%:*}; envs=${v#*:}
  env RH_DEBUG=8 $envs timeout 300 python tools/diag.py case9241pegase > $OUT/diag_$tag.txt 2>&1
  echo "== $tag" >> $OUT/kblk.txt
  python tools/kblk_prof.py gpurun_out/kblk_prof.bin >> $OUT/kblk.txt 2>&1
done
cat $OUT/kblk.txt
