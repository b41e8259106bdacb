#!/bin/bash
# config-2 sweep of the periodic steady-state tolerance (the predictor only feeds guesses)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for r in 1e-8 1e-6 1e-4 1e-3 1e-2; do
  MLMCP_SS_RTOL=$r timeout 300 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$r', d['ms_per_step'], d['detail']['pcg_iterations_per_estimate'], d['detail']['expectation'])"
done | tee gpurun_out/ss_sweep.txt
