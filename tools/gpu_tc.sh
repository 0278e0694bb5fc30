set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tc" > gpurun_out/pytest_tc.log 2>&1; echo t=$?
tail -n 15 gpurun_out/pytest_tc.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --keys tc > gpurun_out/bench_tc.log 2>&1; echo tc=$?
tail -c 1500 gpurun_out/bench_tc.log
