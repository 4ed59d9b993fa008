#!/bin/bash
set -u
O=gpurun_out/${1:-r2b}; mkdir -p $O
timeout 600 python tools/timeline.py --config c3 > $O/timeline_c3.txt 2>&1
timeout 600 python tools/timeline.py --config c2 > $O/timeline_c2.txt 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -q -s -rf --timeout 600 -k "odd or host_io" > $O/pytest_fix.log 2>&1; echo "pytest exit $?" >> $O/pytest_fix.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu && /tmp/fp64_peak > $O/fp64_peak.txt 2>&1
timeout 2400 python -m pytest tests -m "gpu and slow" -q -s -rf --timeout 1800 > $O/pytest_slow.log 2>&1; echo "pytest exit $?" >> $O/pytest_slow.log
echo done > $O/DONE
