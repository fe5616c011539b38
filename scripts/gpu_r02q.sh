bash scripts/gpu_bench_ab.sh r02q '--no-hamming --steps 8 --warmup 3' ';TK_NO_PAIR=1;;TK_NO_PAIR=1' 'tests/test_gpu_parity.py'
