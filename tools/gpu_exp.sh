timeout 300 python tools/vt_probe.py
timeout 300 ncu --metrics gpu__time_duration.sum -k regex:k_vt --launch-skip 50 -c 40 --csv --log-file gpurun_out/vt_launch.csv python tools/vt_probe.py > /dev/null 2>&1; echo ncu=$?
