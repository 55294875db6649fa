#!/bin/bash
# tools/profile.sh TAG LAYOUT KERNEL_REGEX [WORKLOAD] [EXTRA bench.py ARGS] : one `ncu --set full` capture of the headline kernel on the C5 workload
# (bench.py inputs), summarised into gpurun_out/ncu_TAG.txt; plus the launch list of the same command.
TAG=$1; LAYOUT=${2:-pbrt-q16}; K=${3:-chrt2_kernel}; WL=${4:-c5}; EXTRA=${5:-}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:$K --launch-skip 2 --launch-count 1 -f -o gpurun_out/ncu_$TAG \
  python bench.py --workload $WL --layout $LAYOUT --no-e2e --no-cpu --sweep '' --steps 2 --warmup 1 $EXTRA > gpurun_out/ncu_$TAG.log 2>&1
python tools/ncu_summary.py gpurun_out/ncu_$TAG.ncu-rep --sass > gpurun_out/ncu_$TAG.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --workload $WL --layout $LAYOUT --no-e2e --no-cpu --sweep '' --steps 2 --warmup 1 $EXTRA > gpurun_out/launches_$TAG.log 2>&1
head -60 gpurun_out/ncu_$TAG.txt
