bash scripts/gpu_bench_ab.sh r02r '--no-hamming --steps 8 --warmup 3' ';TK_FFG_TWOPASS=1;;TK_FFG_TWOPASS=1' 'tests -m gpu'
