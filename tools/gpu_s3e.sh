#!/bin/bash
# Launch list of the c3 LU-tracked step (where the ~10 ms outside the A-passes go).
set -u
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-s3e}; O=gpurun_out/$TAG; mkdir -p $O
CMD="python bench.py --config c3 --method lu --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks"
if timeout 600 $CMD > $O/plain.log 2>&1; then
  TSSVD_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1
fi
python tools/launch_summary.py $O/launches.csv > $O/launch_summary.txt 2>&1
echo done > $O/DONE
