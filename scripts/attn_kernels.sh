# Attention kernels at the 8B layer shape: parity tests, CUDA-event times, per-kernel ncu times.
timeout 600 python -m pytest tests/test_gpu_attention.py -q -x > gpurun_out/attn_t.log 2>&1; echo "tests exit $?"; tail -1 gpurun_out/attn_t.log
python scripts/attn_probe.py 20
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:attn_ --csv python scripts/attn_probe.py 3 > gpurun_out/attn_k.csv 2>&1
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/attn_k.csv")) if len(r) > 14 and r[0].isdigit()]
d = collections.defaultdict(list)
for r in rows:
    d[(r[4].split("(")[0][-22:], r[12][:28])].append(float(r[14].replace(",", "")))
for k, v in sorted(d.items()):
    print(k, round(sum(v) / len(v), 1))
PY
