# scratch GPU session script (run via gpurun; outputs under gpurun_out/)
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s8_pytest.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/s8_pytest.log
timeout 900 python bench.py > gpurun_out/s8_bench.json 2> gpurun_out/s8_bench.err; echo "bench exit $?"
python -c "
import json;d=json.load(open('gpurun_out/s8_bench.json'));p=d['phases_ms_per_step']
print(round(d['value']), round(d['e2e']['value']), round(d['roofline']['frac'],3), d['adamw'], 'update', p['update'], 'loss', p['loss'], d['clocks'])"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:adamw_f32_bulk -c 1 -o gpurun_out/s8_adamw python tools/probe_adamw.py > gpurun_out/s8_ncu_adamw.log 2>&1; echo "ncu adamw exit $?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:loss_ce_vec -c 1 -o gpurun_out/s8_ce python tools/probe_instep.py > gpurun_out/s8_ncu_ce.log 2>&1; echo "ncu ce exit $?"
