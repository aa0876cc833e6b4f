for i in 1 2; do
for v in cur noprobe; do
L=""; [ "$v" != "cur" ] && L=paper_1504_04804_b200/libmgraph_b200_$v.so
env ${L:+MG_LIB_PATH=$L} timeout 300 python tools/graph_probe.py 26 ref 2>&1 | grep ref | sed "s/^/[$v] /"
done
done
timeout 300 python tools/timeline.py dobfs 26 0 > gpurun_out/tl_ref_src0_c.txt 2>&1
