#!/bin/bash
# Round-end evidence on the final build: GPU suite, smoke, bench lines (default c3, c2, c4, and the
# NEXT-2 / NEXT-4 variants).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 3000 python -m pytest tests -m gpu -q --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config c2 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 python bench.py --config c4 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
timeout 900 python bench.py --config c2 --method tsqr --no-cpu-baseline > $O/bench_c2_tsqr.json 2> $O/bench_c2_tsqr.err
timeout 900 python bench.py --config c3 --method tsqr --no-cpu-baseline > $O/bench_c3_tsqr.json 2> $O/bench_c3_tsqr.err
timeout 900 python bench.py --config c3 --method lu --no-cpu-baseline > $O/bench_c3_lu.json 2> $O/bench_c3_lu.err
