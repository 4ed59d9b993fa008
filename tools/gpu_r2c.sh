#!/bin/bash
set -u
O=gpurun_out/${1:-r2c}; mkdir -p $O
timeout 900 python -m pytest tests -m "gpu and not slow" -q -s -rf --timeout 600 -k "matmul or lowrank" > $O/pytest_sk.log 2>&1; echo "pytest exit $?" >> $O/pytest_sk.log
timeout 900 python tools/bench_diag.py --steps 5 > $O/bench_diag.txt 2>&1
timeout 600 python tools/timeline.py --config c3 > $O/timeline_c3_sk.txt 2>&1
TSSVD_NN_SK=0 timeout 600 python tools/timeline.py --config c3 > $O/timeline_c3_nosk.txt 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"gemm_nn_kernel|gemm_tn_kernel" -c 2 -o $O/c3prof python tools/profile_step.py --config c3 --steps 1 > $O/ncu_c3.log 2>&1
python tools/ncu_summary.py $O/c3prof.ncu-rep > $O/c3_ncu_full_summary.txt 2>&1
TSSVD_NN_SK=0 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"gemm_nn_kernel" -c 1 -o $O/c3prof_nosk python tools/profile_step.py --config c3 --steps 1 > $O/ncu_c3_nosk.log 2>&1
python tools/ncu_summary.py $O/c3prof_nosk.ncu-rep > $O/c3_nosk_ncu_full_summary.txt 2>&1
find $O -name '*.ncu-rep' -size +30M -delete
echo done > $O/DONE
