timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo t=$?
tail -n 3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-prefill > gpurun_out/bench_q.log 2>&1; echo b=$?
grep -o '"ms_per_step": [0-9.]*\|"kernel_ms": [0-9.]*\|"e2e": {"value": [0-9.e+]*' gpurun_out/bench_q.log
