#!/bin/bash
# DRAM bytes + duration of ONE recompute GEMM launch (OPT-30B width, n ACT rows)
# per raster / kernel / L2-policy setting, under ncu (cold L2 per launch, clocks
# not locked). GNS > 0 selects the weight-stationary raster (HC_GEMM_GROUP_N).
#   FUSED="1 0" PAIR="1 0" GMS="8 16 32" GNS="0" L2S="0 1" bash scripts/gemm_dram_sweep.sh [n] [model]
n=${1:-122880}
model=${2:-opt-30b}
for fused in ${FUSED:-1 0}; do for pair in ${PAIR:-1 0}; do for g in ${GMS:-8 16 32 64}; do for gn in ${GNS:-0}; do
for l2 in ${L2S:-0 1}; do
  out=$(HC_FUSED_RECOMPUTE=$fused HC_GEMM_PAIR=$pair HC_GEMM_GROUP_M=$g HC_GEMM_GROUP_N=$gn HC_GEMM_L2HINT=$l2 \
    ncu --clock-control none \
        --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct \
        -k regex:gemm --launch-skip 1 -c 1 --csv python scripts/gemm_one.py $n $model 2>/dev/null | grep -v '^==' | tail -5 \
    | awk -F'","' '{gsub(/"/,"",$NF); printf "%s=%s ", $(NF-2), $NF}')
  echo "fused=$fused pair=$pair group_m=$g group_n=$gn l2=$l2 $out"
done; done; done; done; done
