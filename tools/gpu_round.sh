#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list, ncu full capture of the top kernels.
# usage: tools/gpu_round.sh <tag> [bench args...]
set -x
TAG=${1:-r01}; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/gpu.txt
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.txt 2>&1
timeout 900 python bench.py "$@" > $OUT/bench.json 2> $OUT/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 450 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline "$@" > $OUT/ncu_launch_bench.log 2>&1
python tools/launch_summary.py $OUT/launches.csv > $OUT/launch_summary.txt 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_blk|k_for|k_sep_gemm|k_sep_gather|k_muladd" -s 10 -c 8 \
    -o $OUT/prof_hvp python tools/prof_hvp.py case9241pegase 1024 3 > $OUT/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_fact_blocks|k_sep_inverse' -c 4 \
    -o $OUT/prof_fact python tools/prof_hvp.py case9241pegase 64 1 > $OUT/ncu_full_fact.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_chol' -s 6 -c 2 \
    -o $OUT/prof_chol python tools/chol_prof.py 1444 > $OUT/ncu_full_chol.log 2>&1
python tools/ncu_summary.py $OUT/prof_chol.ncu-rep > $OUT/ncu_chol_summary.txt 2>&1
python tools/ncu_summary.py $OUT/prof_hvp.ncu-rep > $OUT/ncu_hvp_summary.txt 2>&1
python tools/ncu_summary.py $OUT/prof_fact.ncu-rep > $OUT/ncu_fact_summary.txt 2>&1
ls -la $OUT
