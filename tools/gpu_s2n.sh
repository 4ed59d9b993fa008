#!/bin/bash
# c3 step-time anomalies (step - sum of pass times up to 10 ms): is the nvidia-smi sampler stalling the host?
cd $GRAFT_REPO_ROOT
O=gpurun_out/s2n; mkdir -p $O
for i in 1 2 3; do
timeout 600 python bench.py --no-e2e --no-cpu-baseline > $O/bench_c3_clk$i.json 2> $O/bench_c3_clk$i.err
timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-clocks > $O/bench_c3_noclk$i.json 2> $O/bench_c3_noclk$i.err
done
echo done > $O/DONE
