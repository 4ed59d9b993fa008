#!/bin/bash
# alpha pass: compile-time K chunk + incremental stage cursor vs runtime KC (A/B in one build)
cd $GRAFT_REPO_ROOT
O=gpurun_out/s2d; mkdir -p $O
for i in 1 2; do
TSSVD_NN_KCT=0 timeout 300 python tools/nn_bench.py nn 200000 20000 25 >> $O/nn.txt 2>&1
timeout 300 python tools/nn_bench.py nn 200000 20000 25 >> $O/nn.txt 2>&1
done
TSSVD_NN_KCT=0 timeout 300 python tools/nn_bench.py nn 500000 40000 60 >> $O/nn.txt 2>&1
timeout 300 python tools/nn_bench.py nn 500000 40000 60 >> $O/nn.txt 2>&1
timeout 300 python tools/nn_bench.py nn 2000000 100 71 >> $O/nn.txt 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q -k "matmul or lowrank" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err
echo done > $O/DONE
