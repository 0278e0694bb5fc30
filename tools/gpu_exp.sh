timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --keys tc --no-prefill --no-e2e > gpurun_out/bench_exp.log 2>&1; echo rc=$?
grep -o '"kernel_ms": [0-9.]*' gpurun_out/bench_exp.log
