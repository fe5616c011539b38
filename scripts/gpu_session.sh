#!/usr/bin/env bash
# One gpurun session: parity tests, smoke, bench, ncu launch list and captures.
#   gpurun --timeout 2400 -- 'bash scripts/gpu_session.sh [tag] [what]'
# what: all (default) | tests | bench | ncu
set -u
TAG=${1:-r01}
WHAT=${2:-all}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
export PYTHONUNBUFFERED=1
nvidia-smi > "$OUT/nvidia-smi.txt" 2>&1
nproc > "$OUT/host.txt"; lscpu | grep -E 'Model name|^CPU\(s\)' >> "$OUT/host.txt"

if [[ $WHAT == all || $WHAT == tests || $WHAT == quick ]]; then
  timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 \
      python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/sanitizer_smoke.log" 2>&1
  echo "exit=$?" >> "$OUT/sanitizer_smoke.log"
  for tool in racecheck synccheck initcheck; do
    timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 \
        python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/sanitizer_$tool.log" 2>&1
    echo "exit=$?" >> "$OUT/sanitizer_$tool.log"
  done
  timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > "$OUT/pytest_gpu.log" 2>&1
  echo "exit=$?" >> "$OUT/pytest_gpu.log"
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
  echo "exit=$?" >> "$OUT/smoke.log"
fi

if [[ $WHAT == all || $WHAT == bench || $WHAT == quick ]]; then
  timeout 900 python bench.py --steps 20 --warmup 5 > "$OUT/bench.json" 2> "$OUT/bench.err"
  echo "exit=$?" >> "$OUT/bench.err"
  timeout 1200 python bench.py --impl reference --steps ${REF_STEPS:-3} --warmup 1 \
      > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
  timeout 600 python bench.py --workload c4 --steps 2 > "$OUT/bench_c4.json" 2> "$OUT/bench_c4.err"
  # BASELINE.json configs[0] / configs[1] (C1, C2): product and reference arms
  for w in c1 c2; do
    timeout 600 python bench.py --workload $w --steps 10 --warmup 3 > "$OUT/bench_$w.json" 2> "$OUT/bench_$w.err"
    timeout 600 python bench.py --workload $w --impl reference --steps 3 --warmup 1 \
        > "$OUT/bench_ref_$w.json" 2> "$OUT/bench_ref_$w.err"
  done
  # N=2 without a launcher: bench.py re-executes itself under torch.distributed.run;
  # on the one-GPU box both ranks share the device over gloo (CUDA IPC peers)
  TK_FORCE_DEVICE=0 TK_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 2 \
      --warmup 3 > "$OUT/bench_shard2_c5.json" 2> "$OUT/bench_shard2_c5.err"
  echo "exit=$?" >> "$OUT/bench_shard2_c5.err"
fi

if [[ $WHAT == all || $WHAT == hash ]]; then
  # valid-set ingest at C5 scale: timing line + per-kernel ncu metrics (profiles/hash/)
  timeout 600 python scripts/profile_hash.py > "$OUT/hash_time.json" 2> "$OUT/hash_time.err"
  timeout 900 ncu --metrics lts__t_sector_hit_rate.pct,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum \
      --clock-control none --csv -k regex:'hash|valid|scatter|dense|lookup' \
      python scripts/profile_hash.py --once > "$OUT/hash_ncu.csv" 2> "$OUT/hash_ncu.err"
  echo "exit=$?" >> "$OUT/hash_ncu.err"
fi

if [[ $WHAT == ref ]]; then
  timeout 1200 python bench.py --impl reference --steps ${REF_STEPS:-3} --warmup 1 \
      > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
  echo "exit=$?" >> "$OUT/bench_ref.err"
fi

if [[ $WHAT == ab ]]; then
  # A/B of build variants (paper_2210_01465_b200/build.py VARIANTS) on the bench workload
  timeout 600 python bench.py --no-cpu --steps 5 > "$OUT/bench_base.json" 2> "$OUT/bench_base.err"
  for v in ${VARIANTS:-t256}; do
    TK_LIB=paper_2210_01465_b200/libtk_landscape_$v.so timeout 600 python bench.py --no-cpu \
        --steps 5 > "$OUT/bench_$v.json" 2> "$OUT/bench_$v.err"
  done
fi

if [[ $WHAT == all || $WHAT == ncu || $WHAT == quick ]]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 3 --no-cpu \
      > "$OUT/ncu_launches.log" 2>&1
  echo "exit=$?" >> "$OUT/ncu_launches.log"
  timeout 900 ncu --set full --clock-control none --import-source on \
      -k regex:ffg_ -s 3 -c 1 -o "$OUT/prof_ffg" \
      python bench.py --steps 1 --warmup 3 --no-cpu > "$OUT/ncu_ffg.log" 2>&1
  echo "exit=$?" >> "$OUT/ncu_ffg.log"
  timeout 1200 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis \
      --section LaunchStats --section Occupancy --section WarpStateStats --section SourceCounters \
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
      --clock-control none --import-source on \
      -k regex:pagerank -s 3 -c 1 -o "$OUT/prof_pr" \
      python bench.py --steps 1 --warmup 3 --no-cpu > "$OUT/ncu_pr.log" 2>&1
  echo "exit=$?" >> "$OUT/ncu_pr.log"
fi
ls -la "$OUT"

if [[ $WHAT == breakdown ]]; then
  bash scripts/ncu_breakdown.sh "$TAG" pagerank c5
  bash scripts/ncu_breakdown.sh "$TAG" ffg_count c5
  TK_LIB=paper_2210_01465_b200/libtk_landscape_t256.so timeout 600 python bench.py --no-cpu \
      --steps 5 > "$OUT/bench_t256.json" 2> "$OUT/bench_t256.err"
fi

if [[ $WHAT == probe ]]; then
  # quick probes: staged-kernel residency of the variants, Hamming C5 bench line
  for v in "" _t256; do
    TK_DEBUG=1 TK_LIB=paper_2210_01465_b200/libtk_landscape$v.so timeout 300 python bench.py \
        --no-cpu --steps 2 --workload c3 > "$OUT/probe$v.json" 2> "$OUT/probe$v.err"
  done
  timeout 900 python bench.py --no-cpu --steps 3 --kind hamming > "$OUT/bench_hamming.json" \
      2> "$OUT/bench_hamming.err"
fi
