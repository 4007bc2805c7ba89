# scratch GPU session script (run via gpurun; outputs under gpurun_out/)
set -x
timeout 600 python -m pytest tests/test_gpu_linear.py -x -q -k "adamw or softmax" > gpurun_out/s4_pytest.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/s4_pytest.log
for k in reg bulk; do CFT_ADAMW_KERNEL=$k timeout 120 python tools/probe_adamw.py; done > gpurun_out/s4_adamw.log 2>&1; cat gpurun_out/s4_adamw.log
B="python bench.py --steps 30 --no-cpu-baseline --no-sweep --no-e2e"
summ='import json,sys;d=json.load(open(sys.argv[1]));p=d["phases_ms_per_step"];print(sys.argv[1],round(d["value"]),"adamw",round(d["adamw"]["GBps_in_step"]),"update",round(p["update"],3),"loss",round(p["loss"],3),"stats",round(p["stats"],3),d["clocks"]["sm_mhz"])'
CFT_ADAMW_KERNEL=reg CFT_CE_KERNEL=vec timeout 600 $B > gpurun_out/s4_old.json 2>gpurun_out/s4_old.err; python -c "$summ" gpurun_out/s4_old.json
timeout 600 $B > gpurun_out/s4_new.json 2>gpurun_out/s4_new.err; python -c "$summ" gpurun_out/s4_new.json
