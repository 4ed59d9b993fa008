#!/bin/bash
# Fourth session, first call: the GPU suite on the rebuilt HEAD library (the multi-rank LU loop
# kernel changed last), smoke, the default bench line (c3), the LU variants, the reference arm.
set -u
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/s4a; mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo "exit $?" >> $O/bench_c3.err
timeout 900 python bench.py --config c3 --method lu --no-cpu-baseline --no-e2e > $O/bench_c3_lu.json 2> $O/bench_c3_lu.err
TSSVD_LU_FUSED=0 timeout 900 python bench.py --config c3 --method lu --no-cpu-baseline --no-e2e > $O/bench_c3_lu_loop.json 2> $O/bench_c3_lu_loop.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 python bench.py --config c2 > $O/bench_c2.json 2> $O/bench_c2.err
echo done > $O/DONE
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
echo done2 > $O/DONE2
