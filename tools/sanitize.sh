#!/bin/bash
# tools/sanitize.sh — compute-sanitizer over the kernels of the tree: memcheck on the all-layout parity probe, racecheck on the
# parity tests (default kernels), the kernel-variant identity tests (treelet / staged / lane-cooperative / two rays per lane), the
# packed-ray entry and the run-time layouts.  Output: gpurun_out/sanitizer.txt
OUT=gpurun_out/sanitizer.txt
mkdir -p gpurun_out
{
echo "compute-sanitizer on B200 ($(git rev-parse --short HEAD 2>/dev/null || echo worktree)): memcheck python tools/gpu_probe.py (all 24 layouts: closest_hit instrumented + plain, closest_point);"
echo "racecheck python -m pytest tests/test_gpu_parity.py -k '<default kernels>' ; racecheck -k '<variants>' ; memcheck tests/test_open_world.py + packed rays"
compute-sanitizer --tool memcheck python tools/gpu_probe.py 2>&1 | grep -E "PARITY|ERROR SUMMARY|mismatch [1-9]" | tail -5
compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -q -x -k "closest_hit_matches_oracle or closest_point_matches_oracle" 2>&1 | grep -E "passed|failed|RACECHECK SUMMARY" | tail -3
compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -q -x -k "lane_cooperative or staged_record or treelet or two_rays or packed" 2>&1 | grep -E "passed|failed|RACECHECK SUMMARY" | tail -3
compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py tests/test_open_world.py -q -x -k "lane_cooperative or staged_record or treelet or two_rays or packed or user_layout or wide_user" 2>&1 | grep -E "passed|failed|ERROR SUMMARY" | tail -3
} > $OUT 2>&1
cat $OUT
