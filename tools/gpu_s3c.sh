#!/bin/bash
# Fused LU elimination: GPU LU tests (incl. bit-identity against the step loop) and the c3 LU
# bench line, fused vs the step loop.  usage: bash tools/gpu_s3c.sh TAG
set -u
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-s3c}; O=gpurun_out/$TAG; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_lu.py -x -q > $O/pytest_lu.log 2>&1; echo "pytest exit $?" >> $O/pytest_lu.log
timeout 900 python bench.py --config c3 --method lu --no-cpu-baseline --no-e2e > $O/bench_c3_lu.json 2> $O/bench_c3_lu.err
TSSVD_LU_FUSED=0 timeout 900 python bench.py --config c3 --method lu --no-cpu-baseline --no-e2e > $O/bench_c3_lu_loop.json 2> $O/bench_c3_lu_loop.err
echo done > $O/DONE
