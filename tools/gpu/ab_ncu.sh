# per-launch ncu metrics of the pull kernels, tiled vs list-based, one source
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,lts__t_sectors.sum
ncu --metrics $M --clock-control none -k regex:"dobfs_pull|frontier_diff" --csv --log-file gpurun_out/ab_tile.csv python tools/dobfs_probe.py 26 0.01 exact ${SRC:-0} > /dev/null 2>&1
MG_PULL_LIST=1 ncu --metrics $M --clock-control none -k regex:"dobfs_pull|frontier_diff" --csv --log-file gpurun_out/ab_list.csv python tools/dobfs_probe.py 26 0.01 exact ${SRC:-0} > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:dobfs_pull_tile -c 1 -o gpurun_out/tile_full python tools/dobfs_probe.py 26 0.01 exact ${SRC:-0} > /dev/null 2>&1
ls -la gpurun_out
