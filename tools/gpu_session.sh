#!/bin/bash
# One gpurun session: GPU tests, bench (c2 + c3), ncu launch list, ncu full capture of the top kernels.
# usage (from the repo root, under gpurun): bash tools/gpu_session.sh [tag]
set -u
TAG=${1:-s}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
python -c "from paper_1612_08709_b200 import build; build.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; echo "exit $?" >> $O/bench_c2.err
if [ "${SKIP_C3:-0}" = 0 ]; then
timeout 1200 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err; echo "exit $?" >> $O/bench_c3.err
fi
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
if timeout 600 $CMD > $O/plain.log 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"syrk|gemm_nn|gemm_tn" -s 30 -c 4 -o $O/prof $CMD > $O/ncu_full.log 2>&1
fi
echo done > $O/DONE
