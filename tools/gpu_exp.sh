for c in 1024 2048 4096; do
CVQ_F2_CHUNK=$c timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-prefill > gpurun_out/bench_exp_$c.log 2>&1; echo "chunk=$c rc=$?"
grep -o '"ms_per_step": [0-9.]*\|"kernel_ms": [0-9.]*' gpurun_out/bench_exp_$c.log
done
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fast_path or bench_shape" > gpurun_out/pt.log 2>&1; echo t=$?; tail -2 gpurun_out/pt.log
