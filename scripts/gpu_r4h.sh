#!/bin/bash
# steady-state solve tolerance sweep (it only feeds guesses): estimate time and PCG iterations
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for tol in 1e-8 1e-6 1e-5 1e-4; do
  MLMCP_SS_RTOL=$tol timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_ss_$tol.log 2> gpurun_out/bench_ss_$tol.err; echo rc=$?
  python - <<PY
import json
d=json.loads(open("gpurun_out/bench_ss_$tol.log").read().strip().splitlines()[-1])
print("$tol", d["ms_per_step"], d["detail"]["pcg_iterations_per_estimate"], d["detail"]["expectation"])
PY
done
