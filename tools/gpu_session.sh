# scratch GPU session script (run via gpurun; outputs under gpurun_out/)
free -g | head -2; nproc
timeout 900 python -m pytest tests/test_gpu_llama.py -q -x > gpurun_out/s24_pytest.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/s24_pytest.log
timeout 900 python bench.py --remat --no-cpu-baseline --no-sweep --no-e2e > gpurun_out/s24_bench_remat.json 2> gpurun_out/s24_bench_remat.err; echo "bench exit $?"
python -c "
import json;d=json.load(open('gpurun_out/s24_bench_remat.json'))
print(round(d['value']), round(d['ms_per_step'],2), d['device_bytes'], d['flat_memory'], d['clocks'])"
