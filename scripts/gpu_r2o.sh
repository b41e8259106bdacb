#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cluster_propagate -s 1 -c 1 -f -o gpurun_out/prof_cluster python scripts/level_times.py 3 > gpurun_out/ncu_cluster.log 2>&1; echo ncu=$?
timeout 900 python scripts/level_breakdown.py 4 3 128 gpurun_out/lb_cfg4_l3.json > gpurun_out/lb_cfg4_l3.log 2>&1; echo lb=$?; grep -v Warn gpurun_out/lb_cfg4_l3.log | tail -18
timeout 900 python scripts/level_breakdown.py 4 0 2048 gpurun_out/lb_cfg4_l0.json > gpurun_out/lb_cfg4_l0.log 2>&1; echo lb0=$?; grep -v Warn gpurun_out/lb_cfg4_l0.log | tail -8
