#!/bin/bash
# tridiagonal QL for Z (fixed: whole-warp shuffles): kernel tests first, then the suite, then timings
cd $GRAFT_REPO_ROOT
O=gpurun_out/s2g; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_ql.py -x -q --timeout=120 > $O/pytest_ql.log 2>&1; rc=$?; echo "exit $rc" >> $O/pytest_ql.log
if [ $rc -ne 0 ]; then echo done > $O/DONE; exit 0; fi
timeout 1200 python -m pytest tests -m "gpu and not slow" -x -q --timeout=300 > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 300 python bench.py --config c2 --no-cpu-baseline --no-e2e > $O/bench_c2.json 2> $O/bench_c2.err
TSSVD_ZEIG=jacobi timeout 300 python bench.py --config c2 --no-cpu-baseline --no-e2e > $O/bench_c2_jac.json 2> $O/bench_c2_jac.err
timeout 600 python bench.py --config c4 --no-cpu-baseline --no-e2e > $O/bench_c4.json 2> $O/bench_c4.err
TSSVD_ZEIG=jacobi timeout 600 python bench.py --config c4 --no-cpu-baseline --no-e2e > $O/bench_c4_jac.json 2> $O/bench_c4_jac.err
echo done > $O/DONE
