#!/bin/bash
# Round-end evidence on the final build (second session): GPU suite (slow included), smoke, bench
# lines (default c3 with cpu_baseline + e2e, reference arm, c2, c4, TSQR / LU variants), the ncu
# launch list of the default bench command, and ncu --set full captures of the c3 and c2 passes.
cd $GRAFT_REPO_ROOT
O=gpurun_out/final4; mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo "exit $?" >> $O/bench_c3.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 python bench.py --config c2 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 python bench.py --config c4 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
timeout 900 python bench.py --config c2 --method tsqr --no-cpu-baseline > $O/bench_c2_tsqr.json 2> $O/bench_c2_tsqr.err
timeout 900 python bench.py --config c3 --method tsqr --no-cpu-baseline --no-e2e > $O/bench_c3_tsqr.json 2> $O/bench_c3_tsqr.err
timeout 900 python bench.py --config c3 --method lu --no-cpu-baseline --no-e2e > $O/bench_c3_lu.json 2> $O/bench_c3_lu.err
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
if timeout 600 $CMD > $O/plain.log 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1
fi
CMD2="python tools/profile_step.py --config c3 --steps 1"
if timeout 900 $CMD2 > $O/plain_c3.log 2>&1; then
  timeout 1500 ncu --set full --clock-control none -k regex:"gemm_nn_kernel|gemm_tn_kernel" -c 2 -o $O/prof_c3 $CMD2 > $O/ncu_full_c3.log 2>&1
  python tools/ncu_summary.py $O/prof_c3.ncu-rep > $O/ncu_full_c3_summary.txt 2>&1
fi
CMD3="python tools/profile_step.py --config c2 --steps 2"
if timeout 600 $CMD3 > $O/plain_c2.log 2>&1; then
  timeout 1200 ncu --set full --clock-control none -k regex:"syrk|gemm_nn|jacobi|tridiag" -s 9 -c 9 -o $O/prof_c2 $CMD3 > $O/ncu_full_c2.log 2>&1
  python tools/ncu_summary.py $O/prof_c2.ncu-rep > $O/ncu_full_c2_summary.txt 2>&1
fi
find $O -name '*.ncu-rep' -size +20M -delete
echo done > $O/DONE
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
echo done2 > $O/DONE2
