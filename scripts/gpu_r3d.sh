#!/bin/bash
# config-4 Parareal level: time per phase (coarse sweeps / fine slices / defects)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/parareal_phases.py 4 16 2>&1 | tail -3 | tee gpurun_out/pr_phases_cfg4.txt
