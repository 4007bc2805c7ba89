# scratch GPU session script (run via gpurun; outputs under gpurun_out/)
timeout 900 python bench.py > gpurun_out/s23_bench.json 2> gpurun_out/s23_bench.err; echo "bench exit $?"
timeout 900 python bench.py --workload llama70b > gpurun_out/s23_bench70b.json 2> gpurun_out/s23_bench70b.err; echo "bench70b exit $?"
timeout 600 python bench.py --workload linear4096 > gpurun_out/s23_bench_linear.json 2> gpurun_out/s23_bench_linear.err; echo "bench linear exit $?"
python tools/gemm_traffic_step.py 30 > /dev/null 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/s23_launches.csv python tools/gemm_traffic_step.py 30 > gpurun_out/s23_traffic.json 2> gpurun_out/s23_ncu.err; echo "ncu exit $?"
