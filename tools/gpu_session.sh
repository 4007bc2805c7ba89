# scratch GPU session script (run via gpurun; outputs under gpurun_out/)
python tools/probe_wgrad_one.py && timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 2 -c 1 -o gpurun_out/s19_wgrad512 python tools/probe_wgrad_one.py > gpurun_out/s19_ncu.log 2>&1; echo "ncu exit $?"
