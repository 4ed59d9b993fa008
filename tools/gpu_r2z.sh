#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_tsqr.py -q -m gpu -x > gpurun_out/r2z_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/r2z_tests.log
timeout 600 python tools/tsqr_time.py c1 c2 c3 > gpurun_out/r2z_time.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_leaf_qr -c 1 -o gpurun_out/r2z_leaf python tools/tsqr_once.py 400000 100 1 > gpurun_out/r2z_ncu.log 2>&1
