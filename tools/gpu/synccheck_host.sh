# synccheck with the device-driven graph loop off (MG_NO_GRAPH=1): every other kernel
MG_NO_GRAPH=1 timeout 1200 compute-sanitizer --print-limit 50 --tool synccheck python tools/sanitize_cases.py > gpurun_out/san_synccheck_hostloop.txt 2>&1
echo "exit $?" >> gpurun_out/san_synccheck_hostloop.txt
tail -n 3 gpurun_out/san_synccheck_hostloop.txt
