#!/bin/bash
# Round profiling recipe (run under gpurun from the repo root): ncu --set full
# captures of each config's dominant kernel, the pull-kernel dram traffic over
# the bench workload, the bench's launch list, then the bench itself.
# Outputs go to gpurun_out/; summaries are copied into profiles/ by hand.
set -x
OUT=gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:dobfs_pull_thread -c 1 -o $OUT/prof_c2_pull_thread python tools/dobfs_probe.py 26 0.01 exact 0 > $OUT/prof_c2.log 2>&1
$NCU -k regex:dobfs_pull_group -c 1 -o $OUT/prof_c2_pull_group python tools/dobfs_probe.py 26 0.01 exact 4301304 >> $OUT/prof_c2.log 2>&1
$NCU -k regex:lb_expand_kernel -s 3 -c 1 -o $OUT/prof_c3_sssp_expand python tools/timeline.py sssp 24 > $OUT/prof_c3.log 2>&1
$NCU -k regex:pr_pull_update_kernel -s 5 -c 1 -o $OUT/prof_c4_pr_pull python tools/timeline.py pr 24 > $OUT/prof_c4.log 2>&1
$NCU -k regex:cc_link_kernel -c 1 -o $OUT/prof_c4_cc_link python tools/timeline.py cc 24 >> $OUT/prof_c4.log 2>&1
$NCU -k regex:"bc_backward_warp|lb_expand" -c 12 -o $OUT/prof_c5_bc python tools/timeline.py bc 24 > $OUT/prof_c5.log 2>&1
# one-page summaries on the box; keep only the pull-thread report (gpurun copies back <= 64 MiB)
for r in $OUT/prof_*.ncu-rep; do python tools/ncu_summary.py $r > ${r%.ncu-rep}.txt; done
find $OUT -name "prof_*.ncu-rep" ! -name "prof_c2_pull_thread.ncu-rep" -delete
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:dobfs_pull --csv --log-file $OUT/pull_traffic.csv python tools/pull_traffic.py > /dev/null 2>&1
python tools/pull_traffic.py --summarise $OUT/pull_traffic.csv > $OUT/pull_traffic.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/bench_under_ncu.log 2>&1
[ -n "$PROFILE_ONLY" ] && exit 0
python bench.py > $OUT/bench.json 2> $OUT/bench.err
python tools/bench_configs.py > $OUT/configs.jsonl 2> $OUT/configs.err
