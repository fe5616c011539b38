mkdir -p gpurun_out/r02t
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pagerank_ham_tiled -c 1 -o gpurun_out/r02t/prof_hamt python bench.py --no-cpu --no-hamming --kind hamming --steps 1 --warmup 0 > gpurun_out/r02t/ncu.log 2>&1
