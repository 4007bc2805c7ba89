# scratch GPU session script (run via gpurun; outputs under gpurun_out/)
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s21_pytest.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/s21_pytest.log
summ='import json,sys;d=json.load(open(sys.argv[1]));p=d["phases_ms_per_step"];print(sys.argv[1],round(d["value"]),round(d["ms_per_step"],2),"e2e",round(d["e2e"]["value"]),"clk",d["clocks"]["sm_mhz"])'
B="python bench.py --no-cpu-baseline --no-sweep"
for r in 1 2; do
CFT_GEMM_PDL=0 timeout 900 $B > gpurun_out/s21_nopdl_$r.json 2>/dev/null; python -c "$summ" gpurun_out/s21_nopdl_$r.json
timeout 900 $B > gpurun_out/s21_pdl_$r.json 2>/dev/null; python -c "$summ" gpurun_out/s21_pdl_$r.json
done
