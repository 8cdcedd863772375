#!/bin/bash
# usage: tools/ncu_launches.sh <tag> <bench args...>   -> gpurun_out/launches_<tag>.csv (+ summary)
tag=$1; shift
python bench.py "$@" > gpurun_out/plain_$tag.json 2> gpurun_out/plain_$tag.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv python bench.py "$@" > gpurun_out/ncu_$tag.log 2>&1
python tools/ncu_summary.py gpurun_out/launches_$tag.csv > gpurun_out/launches_$tag.summary.txt
cat gpurun_out/launches_$tag.summary.txt | head -40
