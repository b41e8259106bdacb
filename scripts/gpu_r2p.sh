#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo tests=$?
grep -E "passed|failed|FAILED" gpurun_out/gputests.log | head -20
timeout 600 python scripts/config_runs.py 3 > gpurun_out/cfg3.jsonl 2>&1; echo cfg3=$?; tail -1 gpurun_out/cfg3.jsonl | cut -c1-330
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cluster_propagate -s 1 -c 1 -f -o gpurun_out/prof_cluster python scripts/level_times.py 3 > gpurun_out/ncu_cluster.log 2>&1; echo ncu=$?
timeout 1500 python scripts/config_runs.py 4 > gpurun_out/cfg4.jsonl 2>&1; echo cfg4=$?; tail -1 gpurun_out/cfg4.jsonl | cut -c1-330
