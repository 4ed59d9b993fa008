#!/bin/bash
# row-tile GEMM passes with compile-time K chunks (28, 52) vs runtime KC; c2 / c4 bench lines
cd $GRAFT_REPO_ROOT
O=gpurun_out/s2k; mkdir -p $O
for i in 1 2; do
for args in "nn 2000000 100 71" "nn 2000000 55 55" "nn 8000000 200 140" "nn 8000000 92 92"; do
  TSSVD_NN_KCT=0 NORMS=1 timeout 300 python tools/nn_bench.py $args >> $O/nn.txt 2>&1
  NORMS=1 timeout 300 python tools/nn_bench.py $args >> $O/nn.txt 2>&1
done
done
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q --timeout=300 -k "matmul or tssvd" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 300 python bench.py --config c2 --no-cpu-baseline --no-e2e > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --config c4 --no-cpu-baseline --no-e2e > $O/bench_c4.json 2> $O/bench_c4.err
echo done > $O/DONE
