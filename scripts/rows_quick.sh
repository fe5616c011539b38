# row-tiled PageRank: parity subset + C5 timing (+ optional ncu)
OUT=gpurun_out/${1:-rowsq}
mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_parity.py -q --timeout 90 -k "row_tiled" -p no:cacheprovider > $OUT/pytest_rows.log 2>&1
echo "exit=$?" >> $OUT/pytest_rows.log
TK_PR_ROWS=1 TK_DEBUG=1 timeout 300 python scripts/pr_once.py c5 3 > $OUT/time.txt 2>&1
for v in ${VARIANTS:-}; do
  echo "== $v" >> $OUT/time.txt
  env $v timeout 300 python scripts/pr_once.py c5 2 >> $OUT/time.txt 2>&1
done
if [[ -n "${NCU:-}" ]]; then
TK_PR_ROWS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:pagerank_rows -c 1 \
   -o $OUT/prof_rows python scripts/pr_once.py c5 1 > $OUT/ncu.log 2>&1
fi
