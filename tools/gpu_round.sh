set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fp16 or long_context or golden" > gpurun_out/pytest_fp16.log 2>&1; echo t=$?
tail -n 3 gpurun_out/pytest_fp16.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-prefill > gpurun_out/bench_c3_fp16.log 2>&1; echo c3=$?
timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-prefill > gpurun_out/bench_c5_fp16.log 2>&1; echo c5=$?
