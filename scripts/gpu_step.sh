mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity_kernels.py -q --timeout 300 > gpurun_out/parity.log 2>&1; echo "parity exit $?"; tail -3 gpurun_out/parity.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?"; tail -3 gpurun_out/bench.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench.json'))
print(round(d['value']), 'tok/s', round(d['ms_per_step'],2), 'ms; e2e', round(d['e2e']['value']), 'step frac', round(d['step_roofline']['frac'],3), 'GEMM frac', round(d['roofline']['frac'],3), d['clocks'])
print('attention', d['attention'])
print({k: round(v,3) for k,v in d['phases_ms_per_step'].items()})
PY
