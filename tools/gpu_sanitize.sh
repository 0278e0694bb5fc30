# compute-sanitizer over the attention kernels at small parity configs
# (tools/sanitize_probe.py); summaries -> gpurun_out/sanitize_*.txt
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 300 python tools/sanitize_probe.py > gpurun_out/sanitize_plain.txt 2>&1; echo plain=$?
for tool in memcheck synccheck racecheck; do
  for part in sp dense fast append; do
    timeout 900 $CS --tool $tool --print-limit 20 python tools/sanitize_probe.py $part > gpurun_out/sanitize_${tool}_${part}.txt 2>&1
    echo "$tool $part rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/sanitize_${tool}_${part}.txt | tail -2 | tr '\n' ' ')"
  done
done
