#!/bin/bash
# Third session: c5 (160 GB, device-built A) bench line on the current kernels, and the default
# c3 line again.  usage: bash tools/gpu_s3b.sh TAG
set -u
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-s3b}; O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 900 python bench.py --config c5 > $O/bench_c5.json 2> $O/bench_c5.err; echo "exit $?" >> $O/bench_c5.err
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo "exit $?" >> $O/bench_c3.err
echo done > $O/DONE
