# For each prebuilt variant (tools/_var/<v>.so): a quick parity subset of the
# tcgen05 tests, then the A/B bench (tools/ab_so.sh).  AB_VARS="a b".
for v in ${AB_VARS}; do
  cp tools/_var/$v.so paper_2506_18879_b200/libcvq_b200.so
  timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_tc_precision.py -q -x -k "sparse_tc or tc_long or bench_scale or tc_2bit or trained or tile_boundaries or mha" > gpurun_out/abchk_$v.log 2>&1
  echo "$v parity: $(tail -1 gpurun_out/abchk_$v.log)"
done
bash tools/ab_so.sh
