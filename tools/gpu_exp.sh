timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tc" > gpurun_out/pt.log 2>&1; echo t=$?; tail -1 gpurun_out/pt.log
for i in 1 2; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-prefill --no-e2e > gpurun_out/b.log 2>&1
echo "$(grep -o '"ms_per_step": [0-9.]*\|"kernel_ms": [0-9.]*' gpurun_out/b.log | tr '\n' ' ')"
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_tc_score" --launch-skip 3 -c 2 --csv --log-file gpurun_out/tc_launch.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-prefill > /dev/null 2>&1
grep -o '"[0-9]*"$' gpurun_out/tc_launch.csv | head -2
