#!/bin/bash
# DRAM traffic per launch of the dominant kernels at the bench's config-3 scale
# (one ncu --set full capture each; numbers land in profiles/traffic_cfg3.json
# via tools/traffic_json.py).  Run under gpurun after a plain bench run.
O=gpurun_out/traffic
mkdir -p $O
python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $O/plain.json 2> $O/plain.err && \
ncu --set full --clock-control none --import-source on --graph-profiling node -k regex:"k_backward_points|k_gather|k_scatter_emit" \
    -s 3 -c 3 -o $O/cfg3 python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --graph off > $O/ncu.log 2>&1
