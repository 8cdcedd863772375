#!/bin/bash
# usage: tools/capture_round.sh <tag>  -- bench line, ncu launch list and ncu --set full of the sweep/factor kernels
tag=$1
python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err || { tail -20 gpurun_out/bench_$tag.err; exit 1; }
cat gpurun_out/bench_$tag.json
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_$tag.json 2> gpurun_out/plain_$tag.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_$tag.log 2>&1
python tools/ncu_summary.py gpurun_out/launches_$tag.csv > gpurun_out/launches_$tag.summary.txt; head -12 gpurun_out/launches_$tag.summary.txt
ncu --set full --clock-control none --import-source on -k regex:'k_(fwd|bwd)_(persist|tiny|top)|k_factor_(persist|tiny)|k_condense|k_kaug_residual|k_g_spmv|k_gt_spmv' -s 0 -c 24 \
    -o gpurun_out/prof_$tag python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_$tag.log 2>&1
tail -2 gpurun_out/ncu_full_$tag.log
