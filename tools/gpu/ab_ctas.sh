# expansion occupancy A/B: DOBFS expansion compiled for 5 (default), 4, 6 CTAs/SM;
# graph loop + reference schedule on the bench sources, SSSP/BC device time
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dense_push.py -x -q -k "dobfs or bfs or sssp or bc or dense" 2>&1 | tail -2
for i in 1 2; do
for v in "" c4 c6; do
L=""; [ -n "$v" ] && L=paper_1504_04804_b200/libmgraph_b200_$v.so
env ${L:+MG_LIB_PATH=$L} timeout 300 python tools/graph_probe.py 26 ref 2>&1 | grep ref | sed "s/^/[$v] /"
env ${L:+MG_LIB_PATH=$L} timeout 300 python tools/graph_probe.py 26 graph 2>&1 | grep graph | sed "s/^/[$v] /"
done
MG_EXPAND_CTAS_PER_SM=6 timeout 300 python tools/graph_probe.py 26 graph 2>&1 | grep graph | sed "s/^/[grid6] /"
done
timeout 300 python tools/timeline.py sssp 24 2>&1 | grep -E "device_ms"
timeout 300 python tools/timeline.py bc 24 2>&1 | grep -E "device_ms"
