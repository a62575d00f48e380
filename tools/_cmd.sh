timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_inputs.py -x -q -p no:cacheprovider > gpurun_out/r02q_pytest.txt 2>&1; tail -3 gpurun_out/r02q_pytest.txt
bash tools/ab_step.sh r02q "base:" 
RH_DEBUG=8192 timeout 300 python tools/prof_hvp.py case9241pegase 1024 2 cartesian > /dev/null 2>&1; python tools/kfor_prof.py gpurun_out/kfor_prof.bin
