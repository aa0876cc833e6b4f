timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dense_push.py -x -q -k "dobfs or bfs or sssp or bc or dense" 2>&1 | tail -2
for i in 1 2; do
for v in cur ldca; do
L=""; [ "$v" != "cur" ] && L=paper_1504_04804_b200/libmgraph_b200_$v.so
env ${L:+MG_LIB_PATH=$L} timeout 300 python tools/graph_probe.py 26 ref 2>&1 | grep ref | sed "s/^/[$v] /"
done
done
timeout 300 python tools/graph_probe.py 26 graph 2>&1 | grep graph | sed "s/^/[cur] /"
