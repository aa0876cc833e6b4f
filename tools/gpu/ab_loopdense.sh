# device loop: dense pushes off (default) vs on (2^20 arcs), end kernel at 4 or 8 CTAs/SM
for i in 1 2; do
timeout 300 python tools/graph_probe.py 26 graph 2>&1 | grep graph | sed "s/^/[off] /"
MG_DOBFS_LOOP_DENSE_ARCS=1048576 timeout 300 python tools/graph_probe.py 26 graph 2>&1 | grep graph | sed "s/^/[on] /"
MG_LIB_PATH=paper_1504_04804_b200/libmgraph_b200_end8.so MG_DOBFS_LOOP_DENSE_ARCS=1048576 timeout 300 python tools/graph_probe.py 26 graph 2>&1 | grep graph | sed "s/^/[on-end8] /"
MG_LIB_PATH=paper_1504_04804_b200/libmgraph_b200_end8.so timeout 300 python tools/graph_probe.py 26 graph 2>&1 | grep graph | sed "s/^/[off-end8] /"
done
