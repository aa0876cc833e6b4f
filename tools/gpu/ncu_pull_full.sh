# ncu --set full of the first pull of source 0 (RMAT-26 exact-cost DOBFS) for
# the word-parallel kernel and the list kernel, source-level
ncu --set full --import-source on --clock-control none -k regex:dobfs_pull_words -c 1 -o gpurun_out/words_full python tools/dobfs_probe.py 26 0.01 exact 0 > /dev/null 2>&1
MG_PULL_LIST=1 ncu --set full --import-source on --clock-control none -k regex:dobfs_pull_thread -c 1 -o gpurun_out/list_full python tools/dobfs_probe.py 26 0.01 exact 0 > /dev/null 2>&1
ls -la gpurun_out
