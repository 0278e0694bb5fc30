set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tc_score -c 1 -f -o gpurun_out/tc_full5 python bench.py --keys tc --steps 1 --warmup 3 --no-cpu-baseline --no-prefill > gpurun_out/ncu_tc.log 2>&1; echo ncu=$?
tail -5 gpurun_out/ncu_tc.log
