#!/bin/bash
# Round-2 evidence: sanitizers, ncu full captures (c3 alpha/beta, c2 passes), launch lists, c5 test
set -u
O=gpurun_out/${1:-r2g}; mkdir -p $O
for T in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $T --print-limit 50 python tools/sanitize_run.py > $O/sanitizer_$T.txt 2>&1
  echo "exit $?" >> $O/sanitizer_$T.txt
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_nn_kernel -c 1 -o $O/c3_alpha python tools/profile_step.py --config c3 --steps 1 > $O/ncu_c3_alpha.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tn_kernel -c 1 -o $O/c3_beta python tools/profile_step.py --config c3 --steps 1 > $O/ncu_c3_beta.log 2>&1
python tools/ncu_summary.py $O/c3_alpha.ncu-rep > $O/c3_ncu_full_summary.txt 2>&1
python tools/ncu_summary.py $O/c3_beta.ncu-rep >> $O/c3_ncu_full_summary.txt 2>&1
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c3_launches.csv $CMD > $O/ncu_c3_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none -k regex:"syrk|gemm_nn|jacobi" -s 8 -c 8 -o $O/c2prof python tools/profile_step.py --config c2 --steps 2 > $O/ncu_c2.log 2>&1
python tools/ncu_summary.py $O/c2prof.ncu-rep > $O/c2_ncu_full_summary.txt 2>&1
CMD2="python bench.py --config c2 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c2_launches.csv $CMD2 > $O/ncu_c2_launch.log 2>&1
timeout 1500 python -m pytest tests -m "gpu and slow" -q -s -rs --timeout 1200 -k c5 > $O/pytest_c5.log 2>&1; echo "pytest exit $?" >> $O/pytest_c5.log
find $O -name '*.ncu-rep' -size +25M -delete
echo done > $O/DONE
