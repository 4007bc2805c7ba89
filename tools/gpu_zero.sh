timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/z_pytest.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/z_pytest.log
timeout 900 python bench.py --no-sweep --no-cpu-baseline > gpurun_out/z_bench.json 2> gpurun_out/z_bench.err; echo "bench exit $?"
python -c "
import json;d=json.load(open('gpurun_out/z_bench.json'));p=d['phases_ms_per_step']
print(round(d['value']), round(d['ms_per_step'],2), 'update', p['update'], 'adamw', d['adamw'], 'fwd_gemm', p['fwd_gemm'], d['clocks'])"
