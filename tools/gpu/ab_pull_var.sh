# same-box A/B of pull variants on the headline workload (graph loop, 8 bench
# sources) + per-launch ncu of the first pull of source 0 for each
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "dobfs" 2>&1 | tail -1
MG_LIB_PATH=paper_1504_04804_b200/libmgraph_b200_$1.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "dobfs" 2>&1 | tail -1
for i in 1 2 3; do
timeout 300 python tools/graph_probe.py 26 graph 2>&1 | grep graph | sed "s/^/[cur] /"
MG_LIB_PATH=paper_1504_04804_b200/libmgraph_b200_$1.so timeout 300 python tools/graph_probe.py 26 graph 2>&1 | grep graph | sed "s/^/[$1] /"
done
M=gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum
MG_NO_GRAPH=1 ncu --metrics $M --clock-control none -k regex:dobfs_pull_thread --csv --log-file gpurun_out/pv_cur.csv python tools/dobfs_probe.py 26 0.01 exact 0 > /dev/null 2>&1
MG_NO_GRAPH=1 MG_LIB_PATH=paper_1504_04804_b200/libmgraph_b200_$1.so ncu --metrics $M --clock-control none -k regex:dobfs_pull_thread --csv --log-file gpurun_out/pv_var.csv python tools/dobfs_probe.py 26 0.01 exact 0 > /dev/null 2>&1
