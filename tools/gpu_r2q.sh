#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/tsqr_once.py 400000 100 1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_leaf_qr -c 1 -o gpurun_out/r2u_leaf python tools/tsqr_once.py 400000 100 1 > gpurun_out/r2u_ncu.log 2>&1
echo "ncu exit $?" >> gpurun_out/r2u_ncu.log
