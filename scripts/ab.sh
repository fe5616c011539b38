#!/usr/bin/env bash
# A/B of library builds on the bench workload:  bash scripts/ab.sh <tag> "<variants>" [bench args]
#   variants: "base" = product build, others = paper_2210_01465_b200/libtk_landscape_<v>.so
set -u
TAG=${1:-ab}; VARS=${2:-base}; shift 2 || true
OUT=gpurun_out/$TAG; mkdir -p "$OUT"
for v in $VARS; do
  L=paper_2210_01465_b200/libtk_landscape.so
  [ "$v" != base ] && L=paper_2210_01465_b200/libtk_landscape_$v.so
  TK_DEBUG=1 TK_LIB=$L timeout 300 python bench.py --no-cpu --steps 5 "$@" > "$OUT/bench_$v.json" 2> "$OUT/bench_$v.err"
  python - "$OUT/bench_$v.json" "$v" <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[1]))
    print(f"{sys.argv[2]:>8}: {d['value']:8.1f} {d['unit']}  pr_ms={d['phases_ms'].get('pagerank_kernel')} "
          f"ffg_ms={d['phases_ms'].get('ffg_build_kernel')} frac={d['roofline']['frac'] if d.get('roofline') else None}")
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
done
