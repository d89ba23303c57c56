#!/bin/bash
# Recompute GEMM at OPT-30B width (n ACT rows, K = 7168, N = 14336): DRAM bytes,
# duration, SM clock, tensor-pipe activity and L2 hit rate per launch vs the
# raster group (HC_GEMM_GROUP_M), 1-SM kernel and CTA-pair kernel, one ncu pass
# each (--clock-control none), plus the isolated CUDA-event timing.
# Raw outputs: gpurun_out/ggs/<kernel>_<group>.{csv,ms}
N=${1:-122880}
D=gpurun_out/ggs
mkdir -p $D
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct
for k in 1sm pair; do
  for g in 8 16 24 32 64; do
    if [ $k = pair ]; then export HC_GEMM_PAIR_MAX_K=8192; else export HC_GEMM_PAIR_MAX_K=0; fi
    export HC_GEMM_GROUP_M=$g
    python scripts/gemm_one.py $N > $D/${k}_${g}.ms 2>&1
    ncu --metrics $M --clock-control none -k regex:gemm_tn --launch-skip 1 -c 1 --csv \
        python scripts/gemm_one.py $N > $D/${k}_${g}.csv 2>&1
  done
done
