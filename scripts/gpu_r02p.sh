mkdir -p gpurun_out/r02p
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pagerank_ring -c 1 -o gpurun_out/r02p/prof_ring python bench.py --no-cpu --no-hamming --steps 1 --warmup 0 > gpurun_out/r02p/ncu.log 2>&1
TK_PR_STAGED=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:pagerank_staged -c 1 -o gpurun_out/r02p/prof_staged python bench.py --no-cpu --no-hamming --steps 1 --warmup 0 > gpurun_out/r02p/ncu_staged.log 2>&1
