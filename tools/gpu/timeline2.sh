for s in 0 8582448; do
  echo "== src $s host loop"; MG_NO_GRAPH=1 python tools/timeline.py dobfs 26 $s exact 2>&1 | grep -A40 "^span"
done
