# round-2 GPU check: all GPU tests, smoke, C++ drop-in harness, short bench
set -x
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo t=$?
tail -n 15 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/smoke.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-prefill > gpurun_out/bench_q.log 2>&1; echo b=$?
grep -o '"ms_per_step": [0-9.]*\|"kernel_ms": [0-9.]*\|"e2e": {"value": [0-9.e+]*\|"append_ms": [0-9.]*' gpurun_out/bench_q.log
for c in c1 c2; do timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-prefill > gpurun_out/bench_$c.log 2>&1; echo $c=$?; grep -o '"ms_per_step": [0-9.]*\|"kernel_ms": [0-9.]*\|"e2e": {"value": [0-9.e+]*, "unit": "KV-tokens/s", "h2d_bytes_per_step": [0-9]*, "d2h_bytes_per_step": [0-9]*, "ms_per_step": [0-9.]*' gpurun_out/bench_$c.log; done
