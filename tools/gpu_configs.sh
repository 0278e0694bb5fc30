for c in c1 c2 c5; do
timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-prefill > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"
grep -o '"value": [0-9.e+]*\|"ms_per_step": [0-9.]*\|"kernel_ms": [0-9.]*\|"frac": [0-9.]*' gpurun_out/bench_$c.log | head -5
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --config c1 --dist-backend gloo --no-cpu-baseline > gpurun_out/bench_c1_2r.log 2>&1; echo "2rank rc=$?"
grep -o '"value": [0-9.e+]*\|"n_gpus": [0-9]*\|"parallelism": "[^"]*"' gpurun_out/bench_c1_2r.log | head -4
