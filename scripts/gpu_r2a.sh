#!/bin/bash
# round-2 GPU call A: full GPU suite (incl. the large-mesh reference goldens),
# the config-2 bench, compute-sanitizer over every kernel family
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo tests=$?
tail -3 gpurun_out/gputests.log
timeout 900 python bench.py --steps 2 --warmup 1 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo bench=$?
tail -c 600 gpurun_out/bench_cfg2.err
TOOLS=memcheck timeout 1500 bash scripts/sanitize.sh
CASES="fused cluster tile coop direct" TOOLS="racecheck synccheck" timeout 1500 bash scripts/sanitize.sh
