for s in 0 8582448; do
  echo "== words src $s"; python tools/timeline.py dobfs 26 $s exact 2>&1 | tail -40
  echo "== list src $s"; MG_PULL_LIST=1 python tools/timeline.py dobfs 26 $s exact 2>&1 | tail -40
done
