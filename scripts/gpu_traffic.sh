# DRAM bytes of the GEMM family over one Llama-3-8B chunk-local step (chunk 30 of K=60), the
# roofline's `traffic` (bench.py reads profiles/r2_gemm_traffic.json).  Plain run first, then ncu.
mkdir -p gpurun_out
python scripts/gemm_traffic_step.py 30 > gpurun_out/traffic_plain.json 2> gpurun_out/traffic_plain.err || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --profile-from-start off --csv --log-file gpurun_out/traffic_ncu.csv \
    python scripts/gemm_traffic_step.py 30 > gpurun_out/traffic_ncu.json 2> gpurun_out/traffic_ncu.err
echo "ncu exit $?"
