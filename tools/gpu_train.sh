timeout 600 python -m pytest tests/test_train_gpu.py tests/test_valtrain_gpu.py -m gpu -q -x -s > gpurun_out/pytest_train.log 2>&1; echo t=$?
grep -E "rel err|passed|failed|Error|assert" gpurun_out/pytest_train.log | head -30
timeout 900 python tools/bench_train.py > gpurun_out/bench_train.log 2>&1; echo bt=$?
tail -c 2000 gpurun_out/bench_train.log
