#!/bin/bash
# Fourth session: SMSP-balanced runs on top of the new Gram addressing, A/B in one call
# (TSSVD_SYRK_EQUAL=1 = equal runs), Gram-touching GPU tests, smoke, c2 / c4 lines.
set -u
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/${1:-s4h}; mkdir -p $O
W="55 82 92 100 128"
for r in 1 2; do
  TSSVD_SYRK_EQUAL=1 timeout 300 python tools/gram_bench.py --m 2000000 --w $W > $O/gram_equal_$r.txt 2>&1
  timeout 300 python tools/gram_bench.py --m 2000000 --w $W > $O/gram_balanced_$r.txt 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 600 -k "gram or tssvd_c1 or c2_reduced or c4_reduced or ragged or odd_n or lowrank_reduced or square or deterministic or c2_full_size or empty_shard" > $O/pytest_gram.log 2>&1; echo "pytest exit $?" >> $O/pytest_gram.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 600 python bench.py --config c2 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 python bench.py --config c4 --no-cpu-baseline --no-e2e > $O/bench_c4.json 2> $O/bench_c4.err
echo done > $O/DONE
