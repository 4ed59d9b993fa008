#!/bin/bash
set -u
O=gpurun_out/${1:-r2d}; mkdir -p $O
NB="timeout 300 python tools/nn_bench.py"
{
$NB nn 200000 20000 25
TSSVD_NN_SK=0 $NB nn 200000 20000 25
TSSVD_NN_KC=20 $NB nn 200000 20000 25
TSSVD_NN_KC=12 $NB nn 200000 20000 25
TSSVD_L2PROMO=128 $NB nn 200000 20000 25
TSSVD_L2PROMO=0 $NB nn 200000 20000 25
$NB tn 200000 20000 25
TSSVD_L2PROMO=128 $NB tn 200000 20000 25
TSSVD_L2PROMO=0 $NB tn 200000 20000 25
$NB gram 2000000 55 100
TSSVD_L2PROMO=256 $NB gram 2000000 55 100
TSSVD_L2PROMO=128 $NB gram 2000000 55 100
$NB gram 2000000 100
$NB nn 2000000 100 71
$NB nn 2000000 55 55
TSSVD_L2PROMO=256 $NB nn 2000000 55 55
$NB nn 500000 40000 60
TSSVD_NN_SK=0 $NB nn 500000 40000 60
} > $O/nn_bench.txt 2>&1
timeout 1200 python bench.py --steps 10 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err; echo "exit $?" >> $O/bench_c3.err
timeout 900 python bench.py --config c2 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err; echo "exit $?" >> $O/bench_c2.err
echo done > $O/DONE
