#!/bin/bash
# Round-2 GPU session A: box facts, GPU tests (fast), smoke, default bench (c3) + c2 line.
set -u
O=gpurun_out/${1:-r2a}; mkdir -p $O
(nvidia-smi; free -g; nproc; lscpu | grep -i "model name") > $O/box.txt 2>&1
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -s -rf --timeout 600 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 1200 python bench.py --steps 5 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err; echo "exit $?" >> $O/bench_c3.err
timeout 900 python bench.py --config c2 > $O/bench_c2.json 2> $O/bench_c2.err; echo "exit $?" >> $O/bench_c2.err
echo done > $O/DONE
