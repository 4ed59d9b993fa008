#!/bin/bash
# Alg. 1/2/7 GPU parity + first timings
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_tsqr.py -x -q -m gpu > gpurun_out/r2m_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/r2m_tests.log
timeout 600 python tools/tsqr_time.py c1 c2 c3 > gpurun_out/r2m_time.log 2>&1
echo "time exit $?" >> gpurun_out/r2m_time.log
