# scratch GPU session script (run via gpurun; outputs under gpurun_out/)
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s14_pytest.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/s14_pytest.log
timeout 600 python tools/probe_instep.py > gpurun_out/s14_instep.log 2>&1; echo "probe exit $?"; cat gpurun_out/s14_instep.log
timeout 900 python bench.py > gpurun_out/s14_bench.json 2> gpurun_out/s14_bench.err; echo "bench exit $?"
python -c "
import json;d=json.load(open('gpurun_out/s14_bench.json'));p=d['phases_ms_per_step']
print(round(d['value']), round(d['e2e']['value']), round(d['roofline']['frac'],3), round(d['adamw']['GBps_in_step']), round(d['adamw']['frac_of_measured_hbm'],3), 'update', p['update'], 'loss', p['loss'], 'stats', p['stats'], d['clocks'])"
