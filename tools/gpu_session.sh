# scratch GPU session script (run via gpurun; outputs under gpurun_out/)
timeout 300 python tools/debug_fusion.py 0 2>&1 | tail -4
for i in 1 2; do timeout 600 python -m pytest tests/test_gpu_llama.py -q -x -k "fusion_bit_identical" > gpurun_out/s17_pytest_$i.log 2>&1; echo "pytest $i exit $?"; tail -1 gpurun_out/s17_pytest_$i.log; done
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s17_pytest.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/s17_pytest.log
timeout 900 python bench.py > gpurun_out/s17_bench.json 2> gpurun_out/s17_bench.err; echo "bench exit $?"
python -c "
import json;d=json.load(open('gpurun_out/s17_bench.json'));p=d['phases_ms_per_step']
print(round(d['value']), round(d['e2e']['value']), round(d['roofline']['frac'],3), round(d['adamw']['GBps_in_step']), round(d['adamw']['frac_of_measured_hbm'],3), 'fwd', p['fwd_gemm'], 'dgrad', p['dgrad'], 'wgrad', p['wgrad'], 'update', p['update'], 'loss', p['loss'], 'stats', p['stats'], d['sliced_dw']['configs1_sweep'], d['clocks'])"
