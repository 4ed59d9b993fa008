#!/bin/bash
set -u
O=gpurun_out/${1:-r2f}; mkdir -p $O
NB="timeout 300 python tools/nn_bench.py"
{
NORMS=1 $NB nn 2000000 100 71
NORMS=1 $NB nn 2000000 55 55 100
$NB nn 2000000 55 55 100
TSSVD_L2PROMO=256 NORMS=1 $NB nn 2000000 55 55 100
$NB nn 200000 20000 25
TSSVD_NN_MI=3 $NB nn 200000 20000 25
TSSVD_NN_MI=2 $NB nn 200000 20000 25
TSSVD_NN_MI=2 TSSVD_NN_KC=20 $NB nn 200000 20000 25
$NB nn 500000 40000 60
} > $O/nn_bench.txt 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x --timeout 600 > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
timeout 600 python bench.py --config c2 --no-cpu-baseline --no-e2e --steps 20 > $O/bench_c2.json 2>&1
timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 10 > $O/bench_c3.json 2>&1
echo done > $O/DONE
