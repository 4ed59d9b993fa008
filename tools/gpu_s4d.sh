#!/bin/bash
# Fourth session: ncu --set full of the Gram kernel alone (w = 55, 100, 200 at m = 2e6) on the final
# build; only the text summaries come back (the reports exceed the 64 MiB return limit).
set -u
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/${1:-s4g}; mkdir -p $O
timeout 300 python tools/gram_bench.py --m 2000000 --w 55 100 200 > $O/plain.log 2>&1 || exit 1
for w in 55 100 200; do
  timeout 600 ncu --set full --clock-control none -k regex:syrk_kernel -s 2 -c 1 -o /tmp/prof_w$w python tools/gram_bench.py --m 2000000 --w $w > $O/ncu$w.log 2>&1
  python tools/ncu_summary.py /tmp/prof_w$w.ncu-rep > $O/summary_w$w.txt 2>&1
  ncu -i /tmp/prof_w$w.ncu-rep --page details --csv 2>/dev/null | grep -E "Duration|Pipe Fp64|Tensor|DRAM Throughput|Issue Slots Busy|Registers Per|Achieved Occupancy|Bank Conflict|Warp Cycles Per Issued|No Eligible|L1/TEX Hit|Mem Busy|Max Bandwidth" > $O/details_w$w.txt
done
echo done > $O/DONE
