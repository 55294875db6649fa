#!/bin/bash
# tools/final_evidence.sh TAG — the evidence set of a round: GPU suite, bench lines (C5 default with the layout sweep, C4, C1, C3,
# the reference arm) and an ncu capture + launch list of the headline kernel; everything into gpurun_out/
TAG=${1:-final}
mkdir -p gpurun_out
( time python -m pytest tests -m gpu -q 2>&1 | tail -4 ) > gpurun_out/${TAG}_gputest.log 2>&1
( time python bench.py > gpurun_out/${TAG}_bench_c5.json 2> gpurun_out/${TAG}_bench_c5.err ) 2> gpurun_out/${TAG}_bench_c5.time
python bench.py --workload c4 > gpurun_out/${TAG}_bench_c4.json 2> gpurun_out/${TAG}_bench_c4.err
python bench.py --workload c1 > gpurun_out/${TAG}_bench_c1.json 2> gpurun_out/${TAG}_bench_c1.err
python bench.py --workload c3 > gpurun_out/${TAG}_bench_c3.json 2> gpurun_out/${TAG}_bench_c3.err
( time python bench.py --impl reference > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err ) 2> gpurun_out/${TAG}_bench_ref.time
tools/profile.sh ${TAG}_c5_q16 pbrt-q16 chrt2_kernel c5 > /dev/null 2>&1
rm -f gpurun_out/*.ncu-rep
cat gpurun_out/${TAG}_gputest.log gpurun_out/${TAG}_bench_c5.time gpurun_out/${TAG}_bench_ref.time
