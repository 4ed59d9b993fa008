#!/bin/bash
# Gram kernel: 64 rows per stage (A/B build) vs 32
cd $GRAFT_REPO_ROOT
O=gpurun_out/s2m; mkdir -p $O
for i in 1 2; do
for args in "gram 2000000 100" "gram 2000000 55 100" "gram 8000000 200" "gram 8000000 92 200" "gram 200000 25 26"; do
  timeout 300 python tools/nn_bench.py $args >> $O/gram.txt 2>&1
  TSSVD_LIB=tools/ab/libtssvd_kr64.so timeout 300 python tools/nn_bench.py $args >> $O/gram.txt 2>&1
done
done
echo done > $O/DONE
