# A/B of prebuilt libcvq variants (tools/_var/<name>.so, built here with
# CVQ_NVCC_EXTRA flag sets): each is copied over the product .so in the GPU
# box's scratch copy and timed with a short bench.  AB_VARS="a b c", AB_ARGS.
for v in ${AB_VARS}; do
  cp tools/_var/$v.so paper_2506_18879_b200/libcvq_b200.so
  for rep in 1 2; do
    timeout 120 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-prefill --no-e2e ${AB_ARGS} > gpurun_out/ab_$v.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]); print('$v', 'kernel_ms %.3f step_ms %.3f mhz %s' % (d['roofline']['kernel_ms'], d['ms_per_step'], d['clocks']['sm_mhz']))" 2>/dev/null || tail -3 gpurun_out/ab_$v.log
  done
done
