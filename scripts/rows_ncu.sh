# ncu capture of one row-tiled PageRank launch on C5 (+ timing lines)
OUT=gpurun_out/${1:-rowsncu}
mkdir -p $OUT
timeout 300 python scripts/pr_once.py c5 3 > $OUT/time.txt 2>&1
TK_PR_ROWS=0 timeout 300 python scripts/pr_once.py c5 2 >> $OUT/time.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:pagerank_rows -c 1 \
   -o $OUT/prof_rows python scripts/pr_once.py c5 1 > $OUT/ncu.log 2>&1
echo "exit=$?" >> $OUT/ncu.log
