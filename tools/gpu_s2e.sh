#!/bin/bash
# beta pass: compile-time KR + incremental cursor A/B; alpha; Gram; bench lines
cd $GRAFT_REPO_ROOT
O=gpurun_out/s2e; mkdir -p $O
for i in 1 2; do
TSSVD_TN_KRT=0 timeout 300 python tools/nn_bench.py tn 200000 20000 25 >> $O/nn.txt 2>&1
timeout 300 python tools/nn_bench.py tn 200000 20000 25 >> $O/nn.txt 2>&1
timeout 300 python tools/nn_bench.py nn 200000 20000 25 >> $O/nn.txt 2>&1
done
timeout 300 python tools/nn_bench.py gram 2000000 100 >> $O/nn.txt 2>&1
timeout 300 python tools/nn_bench.py gram 2000000 55 100 >> $O/nn.txt 2>&1
timeout 300 python tools/nn_bench.py gram 8000000 200 >> $O/nn.txt 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config c2 --no-cpu-baseline --no-e2e > $O/bench_c2.json 2> $O/bench_c2.err
echo done > $O/DONE
