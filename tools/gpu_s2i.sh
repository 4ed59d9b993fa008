#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/s2i; mkdir -p $O
TSSVD_ZEIG=ql timeout 300 python -m pytest tests/test_gpu_ql.py -x -q --timeout=120 > $O/pytest_ql.log 2>&1; rc=$?; echo "exit $rc" >> $O/pytest_ql.log
if [ $rc -ne 0 ]; then echo done > $O/DONE; exit 0; fi
timeout 300 python tools/ql_once.py > $O/ql_time.txt 2>&1
TSSVD_ZEIG=ql timeout 300 python bench.py --config c2 --no-cpu-baseline --no-e2e > $O/bench_c2_ql.json 2> $O/bench_c2_ql.err
timeout 300 python bench.py --config c2 --no-cpu-baseline --no-e2e > $O/bench_c2_jac.json 2> $O/bench_c2_jac.err
TSSVD_ZEIG=ql timeout 600 python bench.py --config c4 --no-cpu-baseline --no-e2e > $O/bench_c4_ql.json 2> $O/bench_c4_ql.err
timeout 600 python bench.py --config c4 --no-cpu-baseline --no-e2e > $O/bench_c4_jac.json 2> $O/bench_c4_jac.err
TSSVD_ZEIG=ql timeout 900 python -m pytest tests -m "gpu and not slow" -x -q --timeout=300 -k "tssvd or lowrank" > $O/pytest_ql_e2e.log 2>&1; echo "exit $?" >> $O/pytest_ql_e2e.log
echo done > $O/DONE
