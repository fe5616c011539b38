mkdir -p gpurun_out/r02u
bash scripts/gpu_bench_ab.sh r02u '--no-hamming --kind hamming --steps 2 --warmup 2' 'TK_HAM_STAGED=1;TK_HAM_STAGED=1 TK_HAM_ORDER=0' 'tests/test_gpu_parity.py -k hamming'
for o in 1 0; do
TK_HAM_STAGED=1 TK_HAM_ORDER=$o timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:pagerank_ham -c 1 --csv python bench.py --no-cpu --no-hamming --kind hamming --steps 1 --warmup 0 > gpurun_out/r02u/ncu_order$o.csv 2>&1
done
