# device-driven graph loop vs host loop on the bench workload, alternating
for i in 1 2 3; do
MG_GRAPH_LOOP=1 timeout 300 python tools/graph_probe.py 26 2>&1 | tail -2
done
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
