# the multi-process device loop: plain, then memcheck / racecheck / initcheck, host loop under memcheck
timeout 300 python tools/sanitize_cases.py --mp-loop 2>&1 | tail -3
timeout 900 compute-sanitizer --target-processes all --tool memcheck --show-backtrace device python tools/sanitize_cases.py --mp-loop > gpurun_out/san_mploop_memcheck.txt 2>&1; echo "memcheck exit $?"
grep -v "Host Frame" gpurun_out/san_mploop_memcheck.txt | head -30
MG_MP_GRAPH_LOOP=0 timeout 900 compute-sanitizer --target-processes all --tool memcheck python tools/sanitize_cases.py --mp-loop > gpurun_out/san_mploop_memcheck_host.txt 2>&1; echo "memcheck host-loop exit $?"; tail -3 gpurun_out/san_mploop_memcheck_host.txt
