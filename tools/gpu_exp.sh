timeout 300 python tools/prefill_probe.py
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_encode_values|k_encode_keys_table" --csv --log-file gpurun_out/pf_launch.csv python tools/prefill_probe.py > /dev/null 2>&1; echo ncu=$?
grep -o 'k_encode[^"]*".*' gpurun_out/pf_launch.csv | awk -F'","' '{print $1, $NF}' | head
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -q -x -k "encode or prefill or golden or 2bit or value" 2>&1 | tail -1
