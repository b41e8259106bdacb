#!/bin/bash
# bench branches other than the default config: SM-resident (1), cluster (3); new chunking test
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in 3; do
  timeout 600 python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_cfg$c.log 2> gpurun_out/bench_cfg$c.err; echo "cfg$c rc=$?"
  tail -1 gpurun_out/bench_cfg$c.log | cut -c1-250
  tail -2 gpurun_out/bench_cfg$c.err
done
timeout 600 python -m pytest tests/test_gpu_mlmc.py -m gpu -q -p no:cacheprovider -k "direct_chunking or estimator" 2>&1 | tail -3
