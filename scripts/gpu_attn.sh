mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attention.py -q -x --timeout 300 > gpurun_out/attn.log 2>&1; echo "attn exit $?"; tail -30 gpurun_out/attn.log
timeout 900 python -m pytest tests/test_gpu_parity_kernels.py tests/test_gpu_llama.py -q --timeout 600 > gpurun_out/parity_llama.log 2>&1; echo "parity/llama exit $?"; tail -15 gpurun_out/parity_llama.log
