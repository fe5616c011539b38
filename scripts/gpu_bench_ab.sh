#!/usr/bin/env bash
# A/B bench lines on one box:  bash scripts/gpu_bench_ab.sh <tag> "<bench args>" "<ENV=a ENV2=b>;<ENV=c>;..." ["<pytest args>"]
set -u
TAG=$1; ARGS=$2; ENVS=${3:-""}; TESTS=${4:-""}
OUT=gpurun_out/$TAG; mkdir -p "$OUT"
export PYTHONUNBUFFERED=1
if [[ -n "$TESTS" ]]; then
  timeout 900 python -m pytest $TESTS -q -p no:cacheprovider -x > "$OUT/pytest.log" 2>&1
  echo "exit=$?" >> "$OUT/pytest.log"
fi
i=0
IFS=';' read -ra VARS <<< "$ENVS"
[[ ${#VARS[@]} -eq 0 ]] && VARS=("")
for v in "${VARS[@]}"; do
  env $v timeout 600 python bench.py --no-cpu $ARGS > "$OUT/bench_$i.json" 2> "$OUT/bench_$i.err"
  echo "$v" > "$OUT/bench_$i.env"; i=$((i+1))
done
