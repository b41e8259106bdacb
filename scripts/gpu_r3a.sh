#!/bin/bash
# re-entry check: GPU suite + config-2 bench at HEAD
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo tests=$?
grep -E "passed|failed|FAILED" gpurun_out/gputests.log | head -20
timeout 1200 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo bench=$?
cut -c1-400 gpurun_out/bench_cfg2.json; tail -c 300 gpurun_out/bench_cfg2.err
