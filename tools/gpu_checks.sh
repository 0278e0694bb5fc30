# GPU test suite against the CVQ_DEVICE_CHECKS build of libcvq_b200 (stage /
# D-buffer protocol tags + bounds checks that trap), the stand-in for
# compute-sanitizer on this pool.  Build it first:
#   CVQ_NVCC_EXTRA=-DCVQ_DEVICE_CHECKS python -m paper_2506_18879_b200.build --force
#   cp paper_2506_18879_b200/libcvq_b200.so tools/_var/checks.so
cp tools/_var/checks.so paper_2506_18879_b200/libcvq_b200.so
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_checks.log 2>&1
echo "device-checks build: rc=$? $(tail -1 gpurun_out/pytest_checks.log)"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-prefill --no-e2e > gpurun_out/bench_checks.log 2>&1
echo "device-checks bench (C3, 8 steps): rc=$?"
