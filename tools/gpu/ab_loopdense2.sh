timeout 900 python -m pytest tests/test_dense_push.py tests/test_gpu_parity.py -x -q -k "dobfs or bfs or dense" 2>&1 | tail -1
for i in 1 2; do
timeout 300 python tools/graph_probe.py 26 graph 2>&1 | grep graph | sed "s/^/[cur] /"
MG_DOBFS_LOOP_DENSE_ARCS=262144 timeout 300 python tools/graph_probe.py 26 graph 2>&1 | grep graph | sed "s/^/[2^18] /"
MG_DOBFS_LOOP_DENSE_ARCS=4194304 timeout 300 python tools/graph_probe.py 26 graph 2>&1 | grep graph | sed "s/^/[2^22] /"
for v in 12 16; do
MG_LIB_PATH=paper_1504_04804_b200/libmgraph_b200_end$v.so timeout 300 python tools/graph_probe.py 26 graph 2>&1 | grep graph | sed "s/^/[end$v] /"
done
done
