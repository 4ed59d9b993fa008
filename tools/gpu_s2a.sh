#!/bin/bash
# Re-entry check: FP64 pipe microbenchmark (DMMA + DFMA concurrency), GPU tests, default bench line.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s2a; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu && timeout 120 /tmp/fp64_peak > $O/fp64_peak.txt 2>&1
timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo "exit $?" >> $O/bench_c3.err
timeout 600 python bench.py --config c2 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
echo done > $O/DONE
