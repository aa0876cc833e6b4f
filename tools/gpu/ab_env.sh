# same-box A/B of the graph loop on the bench workload: default vs env "$1"
for i in 1 2 3; do
timeout 300 python tools/graph_probe.py 26 graph 2>&1 | grep graph
env $1 timeout 300 python tools/graph_probe.py 26 graph 2>&1 | grep graph
done
