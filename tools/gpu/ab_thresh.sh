# host-loop dense threshold sweep (reference schedule) + graph loop and SSSP/BC
# of the current build against the session-start library, same box
for i in 1 2; do
MG_LIB_PATH=paper_1504_04804_b200/libmgraph_b200_old.so timeout 300 python tools/graph_probe.py 26 graph 2>&1 | grep graph | sed "s/^/[old] /"
timeout 300 python tools/graph_probe.py 26 graph 2>&1 | grep graph | sed "s/^/[cur] /"
for a in 1048576 8388608 33554432; do
MG_DOBFS_DENSE_ARCS=$a timeout 300 python tools/graph_probe.py 26 ref 2>&1 | grep ref | sed "s/^/[$a] /"
done
timeout 300 python tools/timeline.py sssp 24 2>&1 | grep -E "device_ms" | sed "s/^/[cur] sssp /"
timeout 300 python tools/timeline.py bc 24 2>&1 | grep -E "device_ms" | sed "s/^/[cur] bc /"
done
