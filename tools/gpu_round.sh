set -x
for dbg in 0 1 2 3; do
CVQ_TC_DBG=$dbg timeout 600 python bench.py --steps 5 --warmup 2 --keys tc --no-cpu-baseline --no-e2e --no-prefill > gpurun_out/bench_tc_dbg$dbg.log 2>&1; echo dbg$dbg=$?
done
