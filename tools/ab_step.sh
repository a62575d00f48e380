#!/bin/bash
# A/B of env knobs on case9241 (step probe, mask only); variants as "tag:ENV=.. ENV=.." arguments
OUT=gpurun_out/${1:-ab}; shift; mkdir -p $OUT
for v in "$@"; do
  tag=${v%%:*}; envs=${v#*:}
  env PROBE_TAG=$tag $envs timeout 300 python tools/step_probe.py --mask-only case9241pegase >> $OUT/ab.txt 2>&1
done
cat $OUT/ab.txt
