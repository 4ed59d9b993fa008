#!/bin/bash
# NVLS multicast probe; source-level ncu of the c3 alpha and beta kernels.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s2b; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/nvls_probe tools/nvls_probe.cu -lcuda && timeout 60 /tmp/nvls_probe > $O/nvls_probe.txt 2>&1
nvidia-smi topo -m > $O/topo.txt 2>&1; nvidia-smi -q | grep -i -A3 "fabric" >> $O/topo.txt 2>&1
timeout 300 python tools/nn_bench.py nn 200000 20000 25 > $O/nn.txt 2>&1
timeout 300 python tools/nn_bench.py tn 200000 20000 25 >> $O/nn.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_nn_kernel -c 1 -o $O/alpha python tools/nn_bench.py nn 200000 20000 25 > $O/ncu_alpha.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tn_kernel -c 1 -o $O/beta python tools/nn_bench.py tn 200000 20000 25 > $O/ncu_beta.log 2>&1
echo done > $O/DONE
