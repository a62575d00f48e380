timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_inputs.py -x -q -p no:cacheprovider > gpurun_out/r02f_pytest.txt 2>&1; tail -3 gpurun_out/r02f_pytest.txt
bash tools/ab_step.sh r02f "base:" "nofmad:RH_NO_FUSED_MULADD=1" "noprio:RH_NO_PRIO=1"
