CVQ_NVCC_EXTRA="-DSP_EXP_TIMING" python -m paper_2506_18879_b200.build --force > /dev/null 2>&1 || echo build failed
timeout 200 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-prefill --no-e2e > gpurun_out/timing.log 2>&1
grep "wait" gpurun_out/timing.log | sort | uniq | head -60
