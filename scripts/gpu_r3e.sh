#!/bin/bash
# Parareal correction fine solves: tests, config-4 phases with / without, cfg4 512^2 parity
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pr_correction.py tests/test_gpu_large_parity.py -m gpu -q -p no:cacheprovider -k "correction or cfg4 or cfg3_finest" > gpurun_out/gputests_corr.log 2>&1; echo tests=$?
grep -E "passed|failed|FAILED|Error|assert" gpurun_out/gputests_corr.log | head -30
MLMCP_PR_CORRECTION=0 timeout 600 python scripts/parareal_phases.py 4 16 2>&1 | tail -1 | tee gpurun_out/pr_phases_cfg4_off.txt | cut -c1-600
MLMCP_PR_CORRECTION=1 timeout 600 python scripts/parareal_phases.py 4 16 2>&1 | tail -1 | tee gpurun_out/pr_phases_cfg4_on.txt | cut -c1-600
