# A/B experiments on the sparse score kernel (compile-time switches; the round-1
# switches SP_EXP_MMA_ONLY / NO_EPI / NO_STTM / NO_AWAIT / TIMING were measured
# and then removed from attn_sp.cu);
# SP_EXPS = comma-separated flag sets, e.g. "-DA,-DA -DB"
IFS=',' read -ra SETS <<< "${SP_EXPS:-}"
[ ${#SETS[@]} -eq 0 ] && SETS=("")
for e in "${SETS[@]}"; do
  CVQ_NVCC_EXTRA="$e" python -m paper_2506_18879_b200.build --force > /dev/null 2>&1 || echo "build failed $e"
  echo "== $e"
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-prefill --no-e2e > gpurun_out/exp.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/exp.log').read().strip().splitlines()[-1]); print('kernel_ms', d['roofline']['kernel_ms'], 'step_ms', d['ms_per_step'])" 2>/dev/null || tail -3 gpurun_out/exp.log
done
