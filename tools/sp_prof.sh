# ncu --set full of the sparse score kernel at C3 (one launch); read with tools/sp_prof.py
timeout 800 ncu --set full --clock-control none --import-source on -k regex:k_sp_score -c 1 -f -o gpurun_out/prof_sp python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-prefill --no-e2e > gpurun_out/ncu_sp.log 2>&1
echo rc=$?
