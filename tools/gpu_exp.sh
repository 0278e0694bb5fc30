for v in 0 1 0 1; do
if [ $v = 1 ]; then export CVQ_F2_NOALIAS=1; else unset CVQ_F2_NOALIAS; fi
timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-prefill --no-e2e > gpurun_out/b.log 2>&1
echo "noalias=$v $(grep -o '"ms_per_step": [0-9.]*\|"kernel_ms": [0-9.]*' gpurun_out/b.log | tr '\n' ' ')"
done
