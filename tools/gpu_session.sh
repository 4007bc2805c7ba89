# scratch GPU session script (run via gpurun; outputs under gpurun_out/)
timeout 900 python -m pytest tests/test_gpu_engine.py -q -k "artifact" > gpurun_out/s26_pytest.log 2>&1; echo "pytest exit $?"; tail -15 gpurun_out/s26_pytest.log
