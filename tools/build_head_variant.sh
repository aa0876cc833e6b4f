#!/bin/bash
# build the library of a git revision (default HEAD) into
# paper_1504_04804_b200/libmgraph_b200_<name>.so for same-box A/B runs
set -e
name=${1:-head}; rev=${2:-HEAD}
wt=$(mktemp -d /tmp/mgwt.XXXX)
git -C "$(dirname "$0")/.." worktree add -f --detach "$wt" "$rev" > /dev/null
(cd "$wt" && python -c "from paper_1504_04804_b200.build import build; build()" > /dev/null)
cp "$wt/paper_1504_04804_b200/libmgraph_b200.so" "$(dirname "$0")/../paper_1504_04804_b200/libmgraph_b200_$name.so"
git -C "$(dirname "$0")/.." worktree remove --force "$wt"
echo "paper_1504_04804_b200/libmgraph_b200_$name.so <- $rev"
