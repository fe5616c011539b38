# sharded contribution-only step: GPU tests, smoke, two ranks sharing the GPU
set -u
OUT=gpurun_out/shardc; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/summary.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?" >> $OUT/summary.txt
TK_FORCE_DEVICE=0 TK_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 \
  --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 \
  --steps 2 --warmup 3 --workload c3 > $OUT/bench_shard2.json 2> $OUT/bench_shard2.err
echo "shard2 rc=$?" >> $OUT/summary.txt
TK_FORCE_DEVICE=0 TK_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 \
  --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 \
  --steps 2 --warmup 3 > $OUT/bench_shard2_c5.json 2> $OUT/bench_shard2_c5.err
echo "shard2 c5 rc=$?" >> $OUT/summary.txt
