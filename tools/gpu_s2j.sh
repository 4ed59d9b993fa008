#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/s2j; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I include -o /tmp/ql_phase tools/ql_phase.cu -Lpaper_1612_08709_b200/lib -ltssvd_b200 -Xlinker -rpath=$PWD/paper_1612_08709_b200/lib > $O/build.log 2>&1
timeout 120 /tmp/ql_phase > $O/ql_phase.txt 2>&1
echo done > $O/DONE
