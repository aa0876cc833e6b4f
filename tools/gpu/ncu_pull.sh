# ncu --set full of the first pull (thread kernel) of sources 0 and 8582448, host loop
for s in 0 8582448; do
MG_NO_GRAPH=1 ncu --set full --import-source on --clock-control none -k regex:dobfs_pull_thread -c 1 -o gpurun_out/pull_$s python tools/dobfs_probe.py 26 0.01 exact $s > /dev/null 2>&1
done
ls gpurun_out/*.ncu-rep
