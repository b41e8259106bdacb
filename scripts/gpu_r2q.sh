#!/bin/bash
# bench line (config 2) + the reference arm, as the driver runs them
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo bench=$?
tail -c 300 gpurun_out/bench_cfg2.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
cut -c1-300 gpurun_out/bench_ref.json; tail -c 300 gpurun_out/bench_ref.err
