timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_train_gpu.py -m gpu -q -x -k "encode or prefill or golden or 2bit or tie or near or train or append or decode" > gpurun_out/pt.log 2>&1; echo t=$?; tail -1 gpurun_out/pt.log
timeout 300 python tools/prefill_probe.py
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_encode_values|k_encode_keys_table" --csv --log-file gpurun_out/pf_launch.csv python tools/prefill_probe.py > /dev/null 2>&1; echo ncu=$?
grep -o 'k_encode[^(]*(' gpurun_out/pf_launch.csv | head -2; grep -o '"[0-9]*"$' gpurun_out/pf_launch.csv | head -2
