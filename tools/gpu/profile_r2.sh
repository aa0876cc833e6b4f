# round-2 profiles: pull-kernel DRAM traffic over the bench workload (host
# loop, ncu metrics pass) and the bench's launch list (gpu__time_duration)
OUT=gpurun_out
MG_NO_GRAPH=1 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:dobfs_pull --csv --log-file $OUT/pull_traffic.csv python tools/pull_traffic.py > /dev/null 2>&1
python tools/pull_traffic.py --summarise $OUT/pull_traffic.csv > $OUT/pull_traffic.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/bench_under_ncu.log 2>&1
echo done
