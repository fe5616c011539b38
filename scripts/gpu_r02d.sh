mkdir -p gpurun_out/r02d
export PYTHONUNBUFFERED=1
timeout 400 python -m pytest tests/test_gpu_parity.py -k "hamming or c3_scale" -q -p no:cacheprovider -x > gpurun_out/r02d/pytest.log 2>&1; echo "exit=$?" >> gpurun_out/r02d/pytest.log
TK_DEBUG=1 timeout 300 python bench.py --no-cpu --steps 3 --warmup 3 --kind hamming > gpurun_out/r02d/bench_ham.json 2> gpurun_out/r02d/bench_ham.err
TK_HAM_TILED=1 timeout 300 python bench.py --no-cpu --steps 3 --warmup 3 --kind hamming > gpurun_out/r02d/bench_ham_tiled.json 2> gpurun_out/r02d/bench_ham_tiled.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:pagerank_ham -c 1 --csv python bench.py --no-cpu --steps 1 --warmup 0 --kind hamming > gpurun_out/r02d/ncu_ham.csv 2> gpurun_out/r02d/ncu_ham.err
