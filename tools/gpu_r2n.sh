#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_tsqr.py -q -m gpu > gpurun_out/r2n_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/r2n_tests.log
timeout 600 python tools/tsqr_time.py c1 c2 c3 > gpurun_out/r2n_time.log 2>&1
echo "time exit $?" >> gpurun_out/r2n_time.log
timeout 600 python tools/tsqr_once.py 2000000 100 1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2n_tsqr_launches.csv python tools/tsqr_once.py 2000000 100 1 > gpurun_out/r2n_ncu.log 2>&1
echo "ncu exit $?" >> gpurun_out/r2n_ncu.log
