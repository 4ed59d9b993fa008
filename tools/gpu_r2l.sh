#!/bin/bash
set -u
O=gpurun_out/${1:-r2l}; mkdir -p $O
NB="timeout 300 python tools/nn_bench.py"
{ for C in 256 192 128 96 64; do $NB nn 1000000 2000 $C; NORMS=1 $NB nn 100000 600 $C; done; } > $O/panel_nn.txt 2>&1
for P in 256 128 96; do TSSVD_WIDE_PANEL=$P timeout 900 python bench.py --config t3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/bench_t3_p$P.json 2>&1; done
timeout 1500 ncu --set full --clock-control none -k regex:"syrk|gemm_nn" -c 2 -o $O/prof_c4 python tools/profile_step.py --config c4 --steps 1 > $O/ncu_c4.log 2>&1
python tools/ncu_summary.py $O/prof_c4.ncu-rep > $O/c4_ncu_full_summary.txt 2>&1
find $O -name '*.ncu-rep' -size +20M -delete
timeout 900 python tools/ooc_time.py > $O/ooc_c3.txt 2>&1
echo done > $O/DONE
