#!/bin/bash
# round-2 GPU call G: kernel-time breakdown of full config-2 / config-4 estimates, per-level times
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/kernel_breakdown.py 2 gpurun_out/breakdown_cfg2.json > gpurun_out/breakdown_cfg2.log 2>&1; echo bd2=$?
cat gpurun_out/breakdown_cfg2.log | tail -25
timeout 1200 python scripts/level_times.py 4 > gpurun_out/level_times4.log 2>&1; echo lt4=$?
tail -12 gpurun_out/level_times4.log
