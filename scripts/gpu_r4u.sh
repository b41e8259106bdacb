#!/bin/bash
# final: reference arm and a second bench run of the committed state
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err; echo ref=$?
tail -1 gpurun_out/bench_ref.log | cut -c1-200
timeout 1200 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo bench=$?
tail -1 gpurun_out/bench.log | cut -c1-300
