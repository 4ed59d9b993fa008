#!/bin/bash
# A/B of the c2 passes: current build vs the NN_OLD_LOOP variant vs the round-1 library
set -u
O=gpurun_out/${1:-r2e}; mkdir -p $O
NB="timeout 300 python tools/nn_bench.py"
for L in "" tools/ab/libtssvd_oldloop.so tools/ab/libtssvd_r1.so; do
  export TSSVD_LIB=$L; [ -z "$L" ] && unset TSSVD_LIB
  echo "=== lib ${L:-current}"
  NORMS=1 $NB nn 2000000 100 71
  NORMS=1 $NB nn 2000000 55 55 100
  $NB nn 2000000 55 55 100
  $NB gram 2000000 55 100
  $NB gram 2000000 100 100
  $NB nn 200000 20000 25
  TSSVD_L2PROMO=256 NORMS=1 $NB nn 2000000 55 55 100
  TSSVD_L2PROMO=256 $NB gram 2000000 55 100
  timeout 600 python bench.py --config c2 --no-cpu-baseline --no-e2e --steps 20 > $O/bench_c2_$(basename ${L:-current}).json 2>/dev/null
  python -c "import json;d=json.load(open('$O/bench_c2_$(basename ${L:-current}).json'));print('bench c2', d['ms_per_step'], d['roofline']['pass_ms_per_step'])"
done > $O/ab.txt 2>&1
echo done > $O/DONE
