#!/bin/bash
# Fourth session: Gram kernel with loop-invariant shared-window addresses (LDS [R + UR]) -- timing
# against the numbers of gpu_s4c.sh (same widths), the Gram-touching GPU tests, c2 / c4 lines.
set -u
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/${1:-s4e}; mkdir -p $O
W="25 55 64 82 92 100 128 160 200 256"
for r in 1 2; do
  timeout 300 python tools/gram_bench.py --m 2000000 --w $W > $O/gram_$r.txt 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 600 -k "gram or tssvd_c1 or c2_reduced or c4_reduced or ragged or odd_n or lowrank_reduced or square or deterministic or c2_full_size or empty_shard" > $O/pytest_gram.log 2>&1; echo "pytest exit $?" >> $O/pytest_gram.log
timeout 600 python bench.py --config c2 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 python bench.py --config c4 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
echo done > $O/DONE
