timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_tc_score|k_fast_value|k_combine" --launch-skip 9 -c 6 --csv --log-file gpurun_out/launches_c3_tc.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-prefill > gpurun_out/ncu_launches.log 2>&1; echo launches=$?
grep -c "gpu__time" gpurun_out/launches_c3_tc.csv
