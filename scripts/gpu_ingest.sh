# valid-set ingest A/B: partitioned (default) vs direct scatter; tests; ncu of the kernels
OUT=gpurun_out/${1:-ingest}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_valid_set.py tests/test_cpp_dropin.py -m gpu -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "exit=$?" >> $OUT/pytest.log
for v in "" "TK_INGEST_DIRECT=1"; do env $v timeout 300 python scripts/profile_hash.py >> $OUT/hash_time.txt 2>&1; echo "[$v]" >> $OUT/hash_time.txt; done
timeout 600 ncu --metrics lts__t_sector_hit_rate.pct,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv -k regex:'bucket|valid|fill_failed' python scripts/profile_hash.py --once > $OUT/hash_ncu.csv 2> $OUT/hash_ncu.err
