#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list, ncu full capture of the top kernel.
# usage: tools/gpu_round.sh <tag> [bench args...]
set -x
TAG=${1:-r01}; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/gpu.txt
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.txt 2>&1
timeout 900 python bench.py "$@" > $OUT/bench.json 2> $OUT/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline "$@" > $OUT/ncu_launch_bench.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_hvp -s 2 -c 1 -o $OUT/prof_hvp \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline "$@" > $OUT/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_refactor -s 1 -c 1 -o $OUT/prof_refactor \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline "$@" > $OUT/ncu_full_refactor.log 2>&1
ls -la $OUT
