for c in 8192 2048 1024 512 8192 2048; do
CVQ_TC_CHUNK=$c timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-prefill --no-e2e > gpurun_out/b.log 2>&1
echo "chunk=$c $(grep -o '"ms_per_step": [0-9.]*\|"kernel_ms": [0-9.]*\|"sm_mhz": [0-9.]*' gpurun_out/b.log | tr '\n' ' ')"
done
