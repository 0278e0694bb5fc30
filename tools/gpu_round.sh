# Round-end evidence run: tests, smoke, default bench + reference arm, the
# launch list of the timed step, one ncu --set full of the score kernel,
# training throughput.  Outputs under gpurun_out/.
set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo t=$?
tail -n 2 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/bench_c3.log 2>&1; echo c3=$?
tail -c 3000 gpurun_out/bench_c3.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
tail -c 400 gpurun_out/bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_sp_score|k_tc_score|k_fast_value|k_combine" --launch-skip 9 -c 6 --csv --log-file gpurun_out/launches_c3_tc.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-prefill > gpurun_out/ncu_launches.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sp_score|k_tc_score" -c 1 -f -o gpurun_out/prof_score_final python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-prefill --no-e2e > gpurun_out/ncu_full.log 2>&1; echo full=$?
timeout 900 python tools/bench_train.py > gpurun_out/bench_train.log 2>&1; echo train=$?
tail -c 1500 gpurun_out/bench_train.log
