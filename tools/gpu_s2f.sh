#!/bin/bash
# tridiagonal QL for Z: kernel tests, end-to-end parity, c2/c4 timing vs the Jacobi solve
cd $GRAFT_REPO_ROOT
O=gpurun_out/s2f; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_ql.py -x -q > $O/pytest_ql.log 2>&1; echo "exit $?" >> $O/pytest_ql.log
timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 600 python bench.py --config c2 --no-cpu-baseline --no-e2e > $O/bench_c2.json 2> $O/bench_c2.err
TSSVD_ZEIG=jacobi timeout 600 python bench.py --config c2 --no-cpu-baseline --no-e2e > $O/bench_c2_jac.json 2> $O/bench_c2_jac.err
timeout 900 python bench.py --config c4 --no-cpu-baseline --no-e2e > $O/bench_c4.json 2> $O/bench_c4.err
TSSVD_ZEIG=jacobi timeout 900 python bench.py --config c4 --no-cpu-baseline --no-e2e > $O/bench_c4_jac.json 2> $O/bench_c4_jac.err
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err
echo done > $O/DONE
