# A/B of the pull variants on the bench workload (8 sources, RMAT-26), then the
# per-launch ncu metrics of one source
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "dobfs" 2>&1 | tail -2
MG_GRAPH_LOOP=1 timeout 300 python tools/graph_probe.py 26 2>&1 | tail -2
MG_PULL_LIST=1 MG_GRAPH_LOOP=1 timeout 300 python tools/graph_probe.py 26 2>&1 | tail -2
MG_LIB_PATH=paper_1504_04804_b200/libmgraph_b200_occ3.so MG_GRAPH_LOOP=1 timeout 300 python tools/graph_probe.py 26 2>&1 | tail -2
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum
ncu --metrics $M --clock-control none -k regex:"dobfs_pull" --csv --log-file gpurun_out/ab_tile.csv python tools/dobfs_probe.py 26 0.01 exact 0 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:dobfs_pull_tile -c 1 -o gpurun_out/tile_full2 python tools/dobfs_probe.py 26 0.01 exact 0 > /dev/null 2>&1
