timeout 1500 python bench.py > gpurun_out/bench12.log 2>&1; echo rc=$? >> gpurun_out/bench12.log
timeout 300 python scripts/prefill_profile.py --batch 32 --layers 2 > gpurun_out/prefill_prof12.log 2>&1
timeout 300 python scripts/prefill_profile.py --batch 32 --layers 2 --arch opt >> gpurun_out/prefill_prof12.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"prefill_flash|scatter_kv|scatter_act|layernorm" -c 4 -o gpurun_out/ncu_prefill12 python scripts/prefill_profile.py --batch 8 --layers 1 --reps 1 --arch opt > gpurun_out/ncu_prefill12.log 2>&1
