timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_inputs.py -x -q -p no:cacheprovider > gpurun_out/r02s_pytest.txt 2>&1; tail -3 gpurun_out/r02s_pytest.txt
bash tools/ab_step.sh r02s "base:"
