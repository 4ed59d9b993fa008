#!/bin/bash
# Fourth session, fourth call: source-level ncu capture of the narrow Gram (w = 55 and w = 100 at
# m = 2e6) -- what bounds it, since the busiest SMSP's DMMA slots do not (gram_smsp_balance_ab.txt).
set -u
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/s4d; mkdir -p $O
CMD="python tools/gram_bench.py --m 2000000 --w 55 100"
timeout 300 $CMD > $O/plain.log 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:syrk_kernel -s 2 -c 1 -o $O/prof_w55 python tools/gram_bench.py --m 2000000 --w 55 > $O/ncu55.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:syrk_kernel -s 2 -c 1 -o $O/prof_w100 python tools/gram_bench.py --m 2000000 --w 100 > $O/ncu100.log 2>&1
for t in w55 w100; do
  python tools/ncu_summary.py $O/prof_$t.ncu-rep > $O/summary_$t.txt 2>&1
  ncu -i $O/prof_$t.ncu-rep --page source --csv --print-source sass > $O/source_sass_$t.csv 2>/dev/null
  ncu -i $O/prof_$t.ncu-rep --page details --csv > $O/details_$t.csv 2>/dev/null
done
echo done > $O/DONE
