#!/bin/bash
# Fourth session: full GPU suite, smoke and the default bench line on the build with the new Gram
# addressing.
set -u
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/${1:-s4f}; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo "exit $?" >> $O/bench_c3.err
echo done > $O/DONE
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
echo done2 > $O/DONE2
