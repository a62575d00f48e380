#!/bin/bash
# Round-2 GPU session: tests (parity stats logged), smoke, bench, launch list,
# ONE complete batch (random W and Cartesian) under ncu --set full + summaries.
# usage: tools/gpu_r02.sh <tag> [bench args...]
TAG=${1:-r02a}; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/gpu.txt
nproc > $OUT/nproc.txt
RH_PARITY_LOG=$PWD/$OUT/parity.jsonl timeout 1500 python -m pytest tests -m gpu -q -rA -s -p no:cacheprovider > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.txt 2>&1
timeout 1200 python bench.py "$@" > $OUT/bench.json 2> $OUT/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 450 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline "$@" > $OUT/ncu_launch_bench.log 2>&1
python tools/launch_summary.py $OUT/launches.csv > $OUT/launch_summary.txt 2>&1
for kind in cartesian random; do
  timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off \
      -o $OUT/prof_$kind python tools/prof_hvp.py case9241pegase 1024 3 $kind > $OUT/ncu_full_$kind.log 2>&1
  python tools/ncu_summary.py $OUT/prof_$kind.ncu-rep > $OUT/ncu_${kind}_summary.txt 2>&1
  python tools/ncu_batch_summary.py $OUT/prof_$kind.ncu-rep case9241pegase 1024 $kind $TAG > $OUT/ncu_${kind}_batch.json 2>&1
done
ls -la $OUT
