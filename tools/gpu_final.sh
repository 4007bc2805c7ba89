timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f_pytest.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/f_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/f_smoke.log 2>&1; echo "smoke exit $?"
timeout 900 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo "bench exit $?"
python -c "
import json;d=json.load(open('gpurun_out/f_bench.json'))
print(round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), 'frac', round(d['roofline']['frac'],3), 'adamw', round(d['adamw']['GBps_in_step']), round(d['adamw']['frac_of_measured_hbm'],3), d['sliced_dw']['configs1_sweep']['1/8']['tflops'], d['clocks'], d['cpu_baseline']['value'])"
timeout 900 python bench.py --workload llama70b > gpurun_out/f_bench70b.json 2> gpurun_out/f_bench70b.err; echo "bench70b exit $?"
python tools/gemm_traffic_step.py 30 > /dev/null 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/f_launches.csv python tools/gemm_traffic_step.py 30 > gpurun_out/f_traffic.json 2> gpurun_out/f_ncu.err; echo "ncu exit $?"
