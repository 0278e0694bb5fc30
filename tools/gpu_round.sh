set -x
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --keys tc"
timeout 600 $CMD > gpurun_out/plain_tc.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tc_score -s 1 -c 1 -o gpurun_out/prof_tc3 $CMD > gpurun_out/ncu_tc.log 2>&1; echo ncu=$?
