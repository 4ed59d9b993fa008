#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_lu.py -q -m gpu > gpurun_out/r2y_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/r2y_tests.log
timeout 600 python tools/tsqr_time.py c3 > gpurun_out/r2y_time.log 2>&1
echo "time exit $?" >> gpurun_out/r2y_time.log
