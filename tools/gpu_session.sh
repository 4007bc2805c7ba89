# Full GPU validation in one gpurun call (outputs under gpurun_out/):
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash tools/gpu_session.sh'
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?"
python -c "
import json;d=json.load(open('gpurun_out/bench.json'))
print(round(d['value']), 'tok/s', round(d['ms_per_step'],2), 'ms; e2e', round(d['e2e']['value']), '; GEMM frac', round(d['roofline']['frac'],3), '; AdamW', round(d['adamw']['GBps_in_step']), 'GB/s', d['clocks'])"
