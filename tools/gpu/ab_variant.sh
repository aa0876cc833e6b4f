# A/B on the bench workload (8 sources, RMAT-26): the default build vs the
# variants named as arguments (libmgraph_b200_<name>.so), then per-launch ncu
# metrics of the default build's pull kernels for sources 0 and 8582448
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_fabric.py -x -q -k "dobfs or bfs" 2>&1 | tail -2
for i in 1 2; do
MG_GRAPH_LOOP=1 timeout 300 python tools/graph_probe.py 26 2>&1 | tail -2
for v in "$@"; do
MG_LIB_PATH=paper_1504_04804_b200/libmgraph_b200_$v.so MG_GRAPH_LOOP=1 timeout 300 python tools/graph_probe.py 26 2>&1 | tail -2
done
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum
for s in 0 8582448; do
ncu --metrics $M --clock-control none -k regex:"dobfs_pull" --csv --log-file gpurun_out/ab_def_$s.csv python tools/dobfs_probe.py 26 0.01 exact $s > /dev/null 2>&1
done
