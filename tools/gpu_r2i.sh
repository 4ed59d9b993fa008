#!/bin/bash
set -u
O=gpurun_out/${1:-r2i}; mkdir -p $O
timeout 1800 python -m pytest tests -m "gpu" -q -rf --timeout 1200 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo "exit $?" >> $O/bench_c3.err
timeout 600 python bench.py --config c2 > $O/bench_c2.json 2> $O/bench_c2.err; echo "exit $?" >> $O/bench_c2.err
timeout 900 python bench.py --config c4 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err; echo "exit $?" >> $O/bench_c4.err
for C in t5 s21 t4 t3; do
  timeout 900 python bench.py --config $C --steps 3 --warmup 2 > $O/bench_$C.json 2> $O/bench_$C.err; echo "exit $?" >> $O/bench_$C.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
echo done > $O/DONE
