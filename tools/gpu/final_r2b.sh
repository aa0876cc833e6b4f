# round-2 (session 7) measurements: full GPU suite, bench N=1, reference arm,
# per-config lines, ncu of the heavy reference-schedule push and of the C3
# SSSP / C5 BC expansions, bench launch list
set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_final.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputest_final.log
python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
python tools/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "configs rc=$?"
NCU="ncu --set full --clock-control none --import-source on"
timeout 600 $NCU -k regex:lb_expand_kernel -s 1 -c 1 -o gpurun_out/prof_push_ref3 python tools/dobfs_probe.py 26 0.01 ref 0 > gpurun_out/prof_push3.log 2>&1
timeout 600 $NCU -k regex:lb_expand_kernel -s 3 -c 1 -o gpurun_out/prof_c3_sssp python tools/timeline.py sssp 24 > gpurun_out/prof_c3.log 2>&1
for r in prof_push_ref3 prof_c3_sssp; do python tools/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/$r.txt 2>&1; done
timeout 300 python tools/timeline.py sssp 24 > gpurun_out/tl_sssp.txt 2>&1
timeout 300 python tools/timeline.py bc 24 > gpurun_out/tl_bc.txt 2>&1
bash tools/gpu/profile_r2.sh
