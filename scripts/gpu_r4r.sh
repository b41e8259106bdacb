#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for d in 6 auto 6 auto; do
  if [ $d = auto ]; then unset MLMCP_BAND_LSDEG; else export MLMCP_BAND_LSDEG=$d; fi
  timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_ls.log 2> gpurun_out/bench_ls.err
  python - <<PY
import json
d=json.loads(open("gpurun_out/bench_ls.log").read().strip().splitlines()[-1])
print("$d", d["ms_per_step"], d["detail"]["pcg_iterations_per_estimate"])
PY
done
