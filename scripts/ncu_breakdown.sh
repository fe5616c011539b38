#!/usr/bin/env bash
# Throughput breakdown of the dominant kernel (which memory unit binds).
#   gpurun -- 'bash scripts/ncu_breakdown.sh <tag> [regex] [workload]'
set -u
TAG=${1:-r01}; RE=${2:-pagerank}; WL=${3:-c5}
OUT=gpurun_out/$TAG; mkdir -p "$OUT"
timeout 1200 ncu --clock-control none -k regex:$RE -s 3 -c 1 \
  --metrics breakdown:gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed,breakdown:sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,l1tex__m_xbar2l1tex_read_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active \
  --csv python bench.py --workload $WL --steps 1 --warmup 3 --no-cpu > "$OUT/breakdown_$RE.csv" 2> "$OUT/breakdown_$RE.err"
echo "exit=$?" >> "$OUT/breakdown_$RE.err"
