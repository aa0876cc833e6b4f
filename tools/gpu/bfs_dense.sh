timeout 1200 python -m pytest tests/test_dense_push.py -x -q 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_fullsize.py -x -q -k "bfs or c2" 2>&1 | tail -2
for i in 1 2; do
timeout 300 python tools/timeline.py bfs 26 2>&1 | grep device_ms | sed "s/^/[on] /"
MG_DOBFS_DENSE_ARCS=0 timeout 300 python tools/timeline.py bfs 26 2>&1 | grep device_ms | sed "s/^/[off] /"
done
