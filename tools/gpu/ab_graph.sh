# same-box A/B of the graph loop: default build vs variant $1, alternating
for i in 1 2 3; do
timeout 300 python tools/graph_probe.py 26 graph 2>&1 | grep graph
MG_LIB_PATH=paper_1504_04804_b200/libmgraph_b200_$1.so timeout 300 python tools/graph_probe.py 26 graph 2>&1 | grep graph
done
