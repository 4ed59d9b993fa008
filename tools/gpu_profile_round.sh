#!/bin/bash
# Round evidence: GPU tests, full bench lines (c2 default + c3), ncu launch list
# of the bench command, ncu --set full of the top kernels.  usage: bash tools/gpu_profile_round.sh TAG
set -u
TAG=${1:-r}; O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; echo "exit $?" >> $O/bench_c2.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo "exit $?" >> $O/bench_ref.err
if [ "${SKIP_C3:-0}" = 0 ]; then
timeout 1200 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err; echo "exit $?" >> $O/bench_c3.err
fi
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
if timeout 600 $CMD > $O/plain.log 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1
fi
CMD2="python tools/profile_step.py --config c2 --steps 2"
if timeout 600 $CMD2 > $O/plain2.log 2>&1; then
  timeout 1200 ncu --set full --clock-control none -k regex:"syrk|gemm_nn|jacobi" -s 8 -c 8 -o $O/prof $CMD2 > $O/ncu_full.log 2>&1
  python tools/ncu_summary.py $O/prof.ncu-rep > $O/ncu_full_summary.txt 2>&1
fi
echo done > $O/DONE
# c4: full capture of the Gram and GEMM passes (roofline.traffic of `bench.py --config c4`)
if [ "${SKIP_C4:-0}" = 0 ]; then
timeout 900 python bench.py --config c4 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err; echo "exit $?" >> $O/bench_c4.err
CMD3="python tools/profile_step.py --config c4 --steps 1"
timeout 1500 ncu --set full --clock-control none -k regex:"syrk|gemm_nn" -c 2 -o $O/prof_c4 $CMD3 > $O/ncu_full_c4.log 2>&1
python tools/ncu_summary.py $O/prof_c4.ncu-rep > $O/ncu_full_c4_summary.txt 2>&1
fi
# gpurun brings back <= 64 MiB: keep the summaries, drop large reports
find $O -name '*.ncu-rep' -size +20M -delete
echo done2 > $O/DONE2
