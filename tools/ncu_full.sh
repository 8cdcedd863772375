#!/bin/bash
# usage: tools/ncu_full.sh <tag> <kernel regex> <launch-skip> <bench args...>
tag=$1; kre=$2; skip=$3; shift 3
python bench.py "$@" > gpurun_out/plainfull_$tag.json 2> gpurun_out/plainfull_$tag.err && \
ncu --set full --clock-control none --import-source on -k regex:$kre -s $skip -c 1 -o gpurun_out/prof_$tag python bench.py "$@" > gpurun_out/ncufull_$tag.log 2>&1
tail -3 gpurun_out/ncufull_$tag.log
