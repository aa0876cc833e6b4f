for r in 3 2 2.5 3.5 3 4; do
MG_PULL_RATIO=$r timeout 600 python tools/ratio_sweep.py 2>&1 | tail -1 | sed "s/^/[ratio $r] /"
done
