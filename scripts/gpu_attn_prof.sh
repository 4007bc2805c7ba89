mkdir -p gpurun_out
python scripts/attn_probe.py 5 > gpurun_out/attn_probe.log 2>&1 && cat gpurun_out/attn_probe.log &&
ncu --set full --clock-control none --import-source on -k regex:attn_bwd -c 2 -o gpurun_out/attn_prof5 python scripts/attn_probe.py 1 > gpurun_out/attn_ncu.log 2>&1; echo "ncu exit $?"; tail -2 gpurun_out/attn_ncu.log
