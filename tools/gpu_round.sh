set -x
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c3.log 2>&1; echo c3=$?
timeout 600 python bench.py --steps 10 --warmup 3 --keys fp16 --no-cpu-baseline > gpurun_out/bench_c3_fp16.log 2>&1; echo c3h=$?
timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5.log 2>&1; echo c5=$?
timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --keys fp16 > gpurun_out/bench_c5_fp16.log 2>&1; echo c5h=$?
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --keys fp16"
timeout 600 $CMD > gpurun_out/plain2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_fast_score -s 1 -c 1 -o gpurun_out/prof_f1h $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
tail -n 3 gpurun_out/*.log
