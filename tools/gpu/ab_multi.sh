# same-box A/B of the graph loop: default build vs each variant named, alternating, 2 rounds
for i in 1 2; do
echo "default"; timeout 300 python tools/graph_probe.py 26 graph 2>&1 | grep graph
for v in "$@"; do echo "$v"; MG_LIB_PATH=paper_1504_04804_b200/libmgraph_b200_$v.so timeout 300 python tools/graph_probe.py 26 graph 2>&1 | grep graph; done
done
