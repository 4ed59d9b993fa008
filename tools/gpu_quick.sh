#!/bin/bash
# Quick GPU check: tests + c2 bench (+ optional launch list).  usage: bash tools/gpu_quick.sh TAG [launches]
set -u
TAG=${1:-q}; O=gpurun_out/$TAG; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS:-} > $O/bench.json 2> $O/bench.err; echo "exit $?" >> $O/bench.err
if [ "${2:-}" = launches ]; then
  CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS:-}"
  timeout 600 $CMD > $O/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1
fi
echo done > $O/DONE
