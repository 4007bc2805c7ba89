# scratch GPU session script (run via gpurun; outputs under gpurun_out/)
timeout 900 python -m pytest tests/test_gpu_linear.py tests/test_gpu_bounds.py tests/test_gpu_llama.py -q -x > gpurun_out/s13_pytest.log 2>&1; echo "pytest exit $?"; tail -5 gpurun_out/s13_pytest.log
timeout 600 python tools/probe_wgrad.py > gpurun_out/s13_wgrad.log 2>&1; echo "probe exit $?"; cat gpurun_out/s13_wgrad.log
