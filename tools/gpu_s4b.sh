#!/bin/bash
# Fourth session, second call: default bench line with the clock-adjusted fraction, the ncu launch
# list of the same command on the final build, c4 and the TSQR variants.
set -u
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/s4b; mkdir -p $O
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo "exit $?" >> $O/bench_c3.err
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
if timeout 600 $CMD > $O/plain.log 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1
  python tools/launch_summary.py $O/launches.csv > $O/c3_launch_summary.txt 2>&1
fi
timeout 900 python bench.py --config c4 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
timeout 900 python bench.py --config c3 --method tsqr --no-cpu-baseline --no-e2e > $O/bench_c3_tsqr.json 2> $O/bench_c3_tsqr.err
timeout 900 python bench.py --config c2 --method tsqr --no-cpu-baseline > $O/bench_c2_tsqr.json 2> $O/bench_c2_tsqr.err
echo done > $O/DONE
