for n in 8 4 2; do timeout 900 python bench.py --config 4 --tp-emulate $n --no-cpu-baseline --steps 3 > gpurun_out/tpemu_$n.log 2>&1; echo rc=$? >> gpurun_out/tpemu_$n.log; done
