#!/bin/bash
# Round profile capture on the GPU box (run under gpurun): full GPU tests, the
# default bench line, then (each after its command exited 0 without ncu) the
# ncu launch list of the C4 bench command and one --set full capture of the
# CPRAND kernel. Outputs under gpurun_out/.
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; tail -3 gpurun_out/gputests.log
python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err || exit 1
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err
CMD="python bench.py --config c4 --no-cpu --e2e-steps 0 --steps 5 --warmup 3 --no-c5"
$CMD > gpurun_out/bench_short.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:fused_rand -s 5 -c 1 -o gpurun_out/fused_rand_full -f $CMD > gpurun_out/ncu_full.log 2>&1
ncu -i gpurun_out/fused_rand_full.ncu-rep --page raw --csv > gpurun_out/fused_rand_full_raw.csv 2>/dev/null
ls -la gpurun_out/
