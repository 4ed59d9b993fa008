#!/bin/bash
# ncu --set full of the fused LU elimination (first tall + first small launch of the c3 LU step).
set -u
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-s3f}; O=gpurun_out/$TAG; mkdir -p $O
CMD="python bench.py --config c3 --method lu --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks"
TSSVD_GRAPH=0 timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_lu_fused -c 2 -o $O/prof_lu $CMD > $O/ncu.log 2>&1
python tools/ncu_summary.py $O/prof_lu.ncu-rep > $O/summary.txt 2>&1
ncu -i $O/prof_lu.ncu-rep --page source --csv --print-source sass > $O/source_sass.csv 2>/dev/null
ncu -i $O/prof_lu.ncu-rep --page details --csv > $O/details.csv 2>/dev/null
echo done > $O/DONE
