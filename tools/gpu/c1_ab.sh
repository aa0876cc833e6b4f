for i in 1 2; do
for v in cur noeager old; do
L=""; [ "$v" != "cur" ] && L=paper_1504_04804_b200/libmgraph_b200_$v.so
env ${L:+MG_LIB_PATH=$L} timeout 300 python tools/c1_probe.py 2>&1 | sed "s/^/[$v] /"
done
done
