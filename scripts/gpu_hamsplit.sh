# Hamming PageRank by dimension groups (tk_hamsplit.cu): parity, sanitizers, C5 timing + launch list
T=${1:-r02hs}
mkdir -p gpurun_out/$T
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "hamming_tiled_pagerank" > gpurun_out/$T/pytest.log 2>&1; echo exit=$? >> gpurun_out/$T/pytest.log
TK_HAM_SPLIT=1 TK_DEBUG=1 timeout 300 python scripts/pr_once.py c5 3 hamming > gpurun_out/$T/once.txt 2>&1
TK_HAM_SPLIT=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:ham_split --csv --log-file gpurun_out/$T/launches.csv python scripts/pr_once.py c5 1 hamming > /dev/null 2>&1
if [ "$2" = "full" ]; then
TK_HAM_SPLIT=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:ham_split --launch-skip 1 --launch-count 4 -o gpurun_out/$T/split4 python scripts/pr_once.py c5 1 hamming > gpurun_out/$T/ncu_full.log 2>&1
fi
TK_HAM_SPLIT=1 timeout 600 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "hamming_tiled_pagerank and split and (radix0 or radix1 or radix2)" > gpurun_out/$T/memcheck.log 2>&1; echo exit=$? >> gpurun_out/$T/memcheck.log
TK_HAM_SPLIT=1 timeout 600 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "hamming_tiled_pagerank and split and (radix0 or radix1)" > gpurun_out/$T/racecheck.log 2>&1; echo exit=$? >> gpurun_out/$T/racecheck.log
