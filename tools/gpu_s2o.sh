#!/bin/bash
# c3 step-time stability after releasing the generator's host A before timing
cd $GRAFT_REPO_ROOT
O=gpurun_out/s2o; mkdir -p $O
for i in 1 2 3 4; do
timeout 900 python bench.py --no-e2e --no-cpu-baseline > $O/bench_c3_$i.json 2> $O/bench_c3_$i.err
done
BENCH_CLOCKS=nvml timeout 900 python bench.py --no-e2e --no-cpu-baseline > $O/bench_c3_nvml.json 2> $O/bench_c3_nvml.err
echo done > $O/DONE
