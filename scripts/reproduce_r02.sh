#!/bin/bash
# Commands behind the round-2 evidence in profiles/ (run on one B200 from the repo root,
# after `python -c "import __graft_entry__ as g; g.build()"`). Each line names its output.
# Numbers under the 1 kW power cap vary a few percent from box to box.
set -e
mkdir -p gpurun_out

# headline bench line (config 3) with every variant -> profiles/r02_bench_opt30b_final.json
python bench.py > gpurun_out/bench.json
# reference arm (unmodified reference library, no product code) -> r02_bench_reference_arm.json
python bench.py --impl reference > gpurun_out/bench_reference.json
# whole generation, every step timed -> r02_full_generation_opt30b_final.json
python bench.py --full-generation > gpurun_out/full_generation.json
# configs 5 and 4 (N = 1) and B = 256 -> r02_bench_opt13b_cfg5.json, r02_bench_opt66b_cfg4.json, r02_bench_opt30b_b256.json
python bench.py --config 5 --no-cpu-baseline > gpurun_out/cfg5.json
python bench.py --config 4 --no-cpu-baseline --no-sweep > gpurun_out/cfg4.json
python bench.py --batch 256 --no-sweep --no-cpu-baseline > gpurun_out/b256.json

# launch lists -> r02_launches_opt30b_L4_final.csv, r02_config2_launches_summary.txt
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_L4.csv \
    python bench.py --steps 2 --warmup 3 --layers 4 --no-sweep --no-cpu-baseline
ncu --profile-from-start off --clock-control none --csv \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size \
    python scripts/config2_ncu.py > gpurun_out/config2_launches.csv

# recompute GEMM: full capture and DRAM sweeps -> r02_ncu_recompute_fused.txt, r02_recompute_dram_sweep.txt
ncu --clock-control none --set full --import-source on -k regex:gemm --launch-skip 1 -c 1 \
    -o gpurun_out/rec_fused_default python scripts/gemm_one.py 122880
FUSED="1 0" PAIR="1 0" GMS="16 32" GNS="0" L2S="0 1" bash scripts/gemm_dram_sweep.sh 122880 > gpurun_out/dram_sweep.txt
python scripts/gemm_sustained.py --width 7168 --grid "pair=0,1;group=16,32;l2=1"   # r02_gemm_sustained_pair_vs_1sm.txt

# weight-streaming decode GEMMs -> r02_decode_gemm_bench.txt, r02_ncu_wstream.txt
python scripts/decode_gemm_bench.py 50 > gpurun_out/decode_gemm_bench.txt
for s in "128 21504 7168 0" "128 7168 28672 0" "128 50272 7168 3"; do
    ncu --clock-control none -k regex:wstream_kernel --launch-skip 3 -c 1 --csv \
        --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed \
        python scripts/gemm_bench_one.py $s 2 5
done

# L2 probes -> r02_l2_probe.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/l2_probe scripts/l2_probe.cu
for mb in 16 32 48 64 80 96 112 128; do
    ncu --metrics dram__bytes_read.sum --csv gpurun_out/l2_probe $mb 4
done

# parity at depth, soak, sanitizer -> r02_depth_parity_opt30b_final.json, r02_soak_fuzz.txt, r02_compute_sanitizer.txt
python scripts/depth_parity.py
python scripts/soak_fuzz.py 1000 400
for t in memcheck racecheck synccheck; do compute-sanitizer --tool $t python scripts/sanitize_smoke.py; done

# the test suites -> r02_pytest_gpu_final.log
python -m pytest tests -m gpu -q
python -m pytest tests -m "not gpu" -q
