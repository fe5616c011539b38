TK_DEBUG=1 bash scripts/gpu_bench_ab.sh r02o '--no-hamming --steps 5 --warmup 3' ';TK_PR_STAGED=1;TK_RING_CHUNK=32;TK_RING_CHUNK=128' 'tests/test_gpu_parity.py -k ring_pagerank'
