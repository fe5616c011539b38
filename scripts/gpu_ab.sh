#!/usr/bin/env bash
# Quick GPU check: parity suite (or a subset) + short bench A/B lines.
#   gpurun -- 'bash scripts/gpu_ab.sh <tag> "<pytest args>" "<ENV=.. ENV2=..>;<ENV=..>"'
set -u
TAG=${1:-ab}; TESTS=${2:-"tests -m gpu"}; ENVS=${3:-""}
OUT=gpurun_out/$TAG; mkdir -p "$OUT"
export PYTHONUNBUFFERED=1
if [[ "$TESTS" != "none" ]]; then
  timeout 1200 python -m pytest $TESTS -q -p no:cacheprovider -x > "$OUT/pytest.log" 2>&1
  echo "exit=$?" >> "$OUT/pytest.log"
fi
i=0
IFS=';' read -ra VARS <<< "$ENVS"
for v in "" "${VARS[@]}"; do
  env $v timeout 600 python bench.py --no-cpu --no-hamming --steps 10 --warmup 3 > "$OUT/bench_$i.json" 2> "$OUT/bench_$i.err"
  echo "$v" > "$OUT/bench_$i.env"; i=$((i+1))
done
