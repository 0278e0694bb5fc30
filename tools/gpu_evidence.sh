# Round-2 evidence run: bench lines for c3 (default) / c1 / c2 / c5, the
# reference arm, ncu launch lists of the timed steps, ncu --set full of the
# step's kernels and of the prefill encoders, and the issue-path
# microbenchmarks.  Everything lands in gpurun_out/; the summaries are copied
# into profiles/ by hand.
set -x
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/ev_pytest_gpu.log 2>&1; echo pytest=$?; tail -n 3 gpurun_out/ev_pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/ev_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/ev_bench_c3.log 2>&1; echo c3=$?
for c in c1 c2 c5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/ev_bench_$c.log 2>&1; echo $c=$?
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ev_bench_ref.log 2>&1; echo ref=$?
# launch lists (per-launch durations, cold-cache / serialised) of 2 timed steps
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_sp_score|k_fast_value|k_combine" --launch-skip 3 -c 6 --csv --log-file gpurun_out/ev_launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-prefill > /dev/null 2>&1; echo l3=$?
for c in c2 c5; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_sp_score|k_fast_value|k_combine" --launch-skip 3 -c 6 --csv --log-file gpurun_out/ev_launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-prefill > /dev/null 2>&1; echo l$c=$?
done
# full captures: score + value + combine of one C3 step
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sp_score|k_fast_value|k_combine" --launch-skip 3 -c 3 -f -o gpurun_out/ev_c3_step python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-prefill > /dev/null 2>&1; echo full3=$?
# prefill encoders (C4 sample)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_encode_keys_table|k_encode_values" -c 2 -f -o gpurun_out/ev_encode python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo fullenc=$?
tools/umma_pred_bench > gpurun_out/ev_umma_pred.txt 2>&1
tools/umma_ws_probe > gpurun_out/ev_umma_ws.txt 2>&1
# decode-step latency split and prefill probe (+ its launch list)
for c in c1 c2 c3; do timeout 300 python tools/decode_probe.py $c 100 > gpurun_out/ev_decode_$c.txt 2>&1; done
timeout 300 python tools/prefill_probe.py > gpurun_out/ev_prefill.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ev_prefill_launches.csv python tools/prefill_probe.py > /dev/null 2>&1; echo pl=$?
timeout 900 python tools/naive_vs_fused.py > gpurun_out/ev_naive_vs_fused.txt 2>&1; echo nvf=$?
