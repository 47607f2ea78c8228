set -x
CMD="python bench.py --config c4 --no-cpu --e2e-steps 0 --steps 5 --warmup 3 --no-c5"
$CMD > gpurun_out/bench_short.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:fused_rand -s 5 -c 1 -o gpurun_out/fused_rand_full -f $CMD > gpurun_out/ncu_full.log 2>&1
ncu -i gpurun_out/fused_rand_full.ncu-rep --page raw --csv > gpurun_out/fused_rand_full_raw.csv 2>/dev/null
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"replica_kernel|stage_copy" --csv --log-file gpurun_out/e2e_kernels.csv python tests/micro/e2e_probe2.py > gpurun_out/ncu_e2e.log 2>&1
tail -2 gpurun_out/bench_short.log | cut -c1-200
