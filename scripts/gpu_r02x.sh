mkdir -p gpurun_out/r02x
TK_PR_RING=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:pagerank_ring -c 1 -o gpurun_out/r02x/prof_ring4 python bench.py --no-cpu --no-hamming --steps 1 --warmup 0 > gpurun_out/r02x/ncu.log 2>&1
