# same-box A/B of library builds (libmgraph_b200_<name>.so; "" = default):
# DOBFS graph loop + reference schedule over the bench sources, SSSP/BC device time
for i in 1 2; do
for v in "$@"; do
L=""; [ "$v" != "cur" ] && L=paper_1504_04804_b200/libmgraph_b200_$v.so
env ${L:+MG_LIB_PATH=$L} timeout 300 python tools/graph_probe.py 26 graph 2>&1 | grep graph | sed "s/^/[$v] /"
env ${L:+MG_LIB_PATH=$L} timeout 300 python tools/graph_probe.py 26 ref 2>&1 | grep ref | sed "s/^/[$v] /"
env ${L:+MG_LIB_PATH=$L} timeout 300 python tools/timeline.py sssp 24 2>&1 | grep -E "device_ms" | sed "s/^/[$v] sssp /"
env ${L:+MG_LIB_PATH=$L} timeout 300 python tools/timeline.py bc 24 2>&1 | grep -E "device_ms" | sed "s/^/[$v] bc /"
done
done
