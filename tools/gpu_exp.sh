timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -q -x -k "encode or prefill or golden or 2bit" > gpurun_out/pt.log 2>&1; echo t=$?; tail -1 gpurun_out/pt.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b.log 2>&1; echo b=$?
grep -o '"token_heads_per_s": [0-9.e+]*\|"c4_projected_s": [0-9.]*' gpurun_out/b.log
