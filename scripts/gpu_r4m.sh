#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python scripts/parareal_phases.py 4 16 2>&1 | tail -1 | tee gpurun_out/pr_phases_cfg4.txt | cut -c1-1500
