timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/ev_pytest_gpu.log 2>&1; echo pytest=$?; tail -n 3 gpurun_out/ev_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/ev_smoke.log
timeout 900 python bench.py > gpurun_out/ev_bench_c3.log 2>&1; echo c3=$?
for c in c1 c2 c5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/ev_bench_$c.log 2>&1; echo $c=$?
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_sp_score|k_fast_value|k_combine" --launch-skip 3 -c 6 --csv --log-file gpurun_out/ev_launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-prefill > /dev/null 2>&1; echo l3=$?
for c in c2 c5; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_sp_score|k_fast_value|k_combine" --launch-skip 3 -c 6 --csv --log-file gpurun_out/ev_launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-prefill > /dev/null 2>&1; echo l$c=$?
done
timeout 400 ncu --set full --import-source on --clock-control none -k regex:k_fast_value -s 3 -c 1 -o gpurun_out/ev_fv_c3 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-prefill --no-e2e > /dev/null 2>&1; echo fv=$?
for c in c1 c3; do timeout 300 python tools/decode_probe.py $c 100 > gpurun_out/ev_decode_$c.txt 2>&1; done
