#!/bin/bash
# ncu --set full of the c3 beta pass (roofline.traffic), on the final build
cd $GRAFT_REPO_ROOT
O=gpurun_out/s2l; mkdir -p $O
CMD2="python tools/profile_step.py --config c3 --steps 1"
timeout 900 $CMD2 > $O/plain_c3.log 2>&1
timeout 1200 ncu --set full --clock-control none -k regex:"gemm_tn_kernel" -c 1 -o $O/prof_c3_beta $CMD2 > $O/ncu_beta.log 2>&1
python tools/ncu_summary.py $O/prof_c3_beta.ncu-rep > $O/ncu_beta_summary.txt 2>&1
timeout 900 python bench.py --no-e2e --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 300 python bench.py --config c2 --no-cpu-baseline --no-e2e > $O/bench_c2.json 2> $O/bench_c2.err
find $O -name '*.ncu-rep' -size +20M -delete
echo done > $O/DONE
