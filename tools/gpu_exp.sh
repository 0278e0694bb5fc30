for k in fp16 tc fp16; do
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --keys $k --no-e2e > gpurun_out/bench_exp_$k.log 2>&1; echo rc=$?
grep -o '"kernel_ms": [0-9.]*\|"token_heads_per_s": [0-9.]*' gpurun_out/bench_exp_$k.log
done
