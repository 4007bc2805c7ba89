# scratch GPU session script (run via gpurun; outputs under gpurun_out/)
echo "auto: $(timeout 300 python tools/probe_wgrad.py)"
echo "streamK: $(CFT_WGRAD_STREAMK=1 timeout 300 python tools/probe_wgrad.py)"
for sp in 1 2 3 4 6 8; do echo "splits $sp: $(CFT_WGRAD_SPLITS=$sp timeout 300 python tools/probe_wgrad.py)"; done
