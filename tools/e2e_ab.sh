#!/bin/bash
# e2e (rh_reduced_hessian_host, pinned buffers) under env variants "tag:ENV=.. ENV=.."
OUT=gpurun_out/${1:-e2eab}; shift; mkdir -p $OUT
for v in "$@"; do
  tag=${v%%:*}; envs=${v#*:}
  echo "== $tag" >> $OUT/e2e.txt
  env $envs timeout 300 python tools/e2e_probe.py 1024 2>&1 | grep "e2e ms" >> $OUT/e2e.txt
done
cat $OUT/e2e.txt
