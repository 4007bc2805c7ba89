# GEMM DRAM bytes over one 8B step with L2 left warm between kernels (ncu --cache-control none:
# the producer-warm operands of the real step count), for the default rasterisation and with
# the long-K group forced to 16.  Plain run first, then ncu.
mkdir -p gpurun_out
python scripts/gemm_traffic_step.py 30 > gpurun_out/traffic_plain.json 2> gpurun_out/traffic_plain.err || exit 1
for g in default 16; do
  if [ "$g" = default ]; then envs=""; else envs="CFT_GEMM_GROUP_LONGK=$g"; fi
  env $envs ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --cache-control none --profile-from-start off --csv \
      --log-file gpurun_out/traffic_warm_$g.csv python scripts/gemm_traffic_step.py 30 \
      > /dev/null 2> gpurun_out/traffic_warm_$g.err
  echo "ncu ($g) exit $?"
done
