# ncu evidence for round 2 (one gpurun call; each ncu after the same command exited 0):
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash scripts/gpu_profiles.sh'
mkdir -p gpurun_out
# 1. launch list of the whole 8B bench run (warm-up + 2 timed steps + the profiled leg)
python bench.py --layers 32 --steps 2 --warmup 3 --no-sweep --no-cpu-baseline --no-e2e > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv \
    --log-file gpurun_out/r2_launches.csv python bench.py --layers 32 --steps 2 --warmup 3 --no-sweep --no-cpu-baseline --no-e2e > gpurun_out/prof_ncu1.log 2>&1; echo "launch list exit $?"
# 2. full captures: attention forward / backward kernels at the 8B layer shape
python scripts/attn_probe.py 3 > gpurun_out/attn_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:attn_ -c 3 -o gpurun_out/r2_attn python scripts/attn_probe.py 1 > gpurun_out/prof_ncu2.log 2>&1; echo "attn full exit $?"
# 3. full capture: the configs[1] 1/8 sliced-dW (stream-K + TMA reduce-add)
python -c "import bench; bench.slice_sweep(0, reps=2)" > gpurun_out/wg_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_2sm -s 3 -c 1 -o gpurun_out/r2_wgrad18 python -c "import bench; bench.slice_sweep(0, reps=2)" > gpurun_out/prof_ncu3.log 2>&1; echo "wgrad full exit $?"
