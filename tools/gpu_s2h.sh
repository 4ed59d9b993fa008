#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/s2h; mkdir -p $O
timeout 300 python tools/ql_once.py > $O/ql_time.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tridiag -c 1 -o $O/ql python tools/ql_once.py > $O/ncu_ql.log 2>&1
echo done > $O/DONE
