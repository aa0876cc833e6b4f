# same-box: session-start library vs the current one under env settings (graph loop)
for i in 1 2; do
MG_LIB_PATH=paper_1504_04804_b200/libmgraph_b200_old.so timeout 300 python tools/graph_probe.py 26 graph 2>&1 | grep graph | sed "s/^/[old] /"
for e in "X=1" "MG_DOBFS_DENSE_ARCS=0" "MG_DOBFS_DENSE_ARCS=16777216" "MG_EXPAND_CTAS_PER_SM=6" "MG_DOBFS_DENSE_ARCS=0 MG_EXPAND_CTAS_PER_SM=6"; do
env $e timeout 300 python tools/graph_probe.py 26 graph 2>&1 | grep graph | sed "s/^/[$e] /"
done
done
