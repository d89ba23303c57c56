set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputests3.log
timeout 300 python scripts/prefill_profile.py --batch 32 --layers 2 > gpurun_out/prefill_prof.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_flash -c 1 -o gpurun_out/ncu_prefill_attn python scripts/prefill_profile.py --batch 8 --layers 1 --reps 1 > gpurun_out/ncu_prefill.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench3.log 2>&1; echo rc=$? >> gpurun_out/bench3.log
timeout 900 python bench.py --config 4 --no-sweep > gpurun_out/cfg4_planner.log 2>&1; echo rc=$? >> gpurun_out/cfg4_planner.log
