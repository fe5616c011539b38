mkdir -p gpurun_out/r02e
export PYTHONUNBUFFERED=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pagerank_ham_staged -c 1 -o gpurun_out/r02e/prof_ham python bench.py --no-cpu --steps 1 --warmup 0 --kind hamming > gpurun_out/r02e/ncu.log 2>&1
echo "exit=$?" >> gpurun_out/r02e/ncu.log
