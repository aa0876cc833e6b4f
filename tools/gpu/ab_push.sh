# same-box A/B of the dense push (DobfsDev::red) on the bench workload:
# reference schedule (host loop) and exact-cost graph loop, on vs off;
# then the DOBFS parity tests
for i in 1 2; do
timeout 300 python tools/graph_probe.py 26 ref 2>&1 | grep ref
MG_DOBFS_DENSE_DIV=0 timeout 300 python tools/graph_probe.py 26 ref 2>&1 | sed 's/^ref/ref-off/' | grep ref
timeout 300 python tools/graph_probe.py 26 graph 2>&1 | grep graph
MG_DOBFS_DENSE_ARCS=0 timeout 300 python tools/graph_probe.py 26 graph 2>&1 | sed 's/^graph/graph-off/' | grep graph
done
for a in 262144 4194304 16777216; do
MG_DOBFS_DENSE_ARCS=$a timeout 300 python tools/graph_probe.py 26 graph 2>&1 | sed "s/^graph/graph-$a/" | grep graph
done
for r in 6 8; do MG_PULL_RATIO=$r timeout 300 python tools/graph_probe.py 26 graph 2>&1 | sed "s/^graph/graph-ratio$r/" | grep graph; done
timeout 900 python -m pytest tests -m gpu -x -q -k "dobfs or bfs or dense" 2>&1 | tail -3
