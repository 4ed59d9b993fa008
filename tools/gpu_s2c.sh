#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/s2c; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/nvls_probe tools/nvls_probe.cu -lcuda && timeout 60 /tmp/nvls_probe > $O/nvls_probe.txt 2>&1
ls -la /dev/nvidia* >> $O/nvls_probe.txt 2>&1; ps aux | grep -i -E "fabric|imex" | grep -v grep >> $O/nvls_probe.txt 2>&1
echo done > $O/DONE
