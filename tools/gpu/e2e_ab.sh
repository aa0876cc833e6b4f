# end-to-end call time (labels into pinned host memory), download variants
for i in 1 2; do
for sp in 0.4 0.5 0.6; do
echo "split $sp serial:  $(MG_D2H_SPLIT=$sp python tools/e2e_probe.py 2>&1 | tail -1)"
echo "split $sp overlap: $(MG_D2H_OVERLAP=1 MG_D2H_SPLIT=$sp python tools/e2e_probe.py 2>&1 | tail -1)"
done
done
