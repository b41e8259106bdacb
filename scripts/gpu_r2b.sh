#!/bin/bash
# round-2 GPU call B: GPU suite with the region-linear tile operator, A/B of the
# tile operator modes, config-2 bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/tile_ab.py 2 1024 32 > gpurun_out/tile_ab2.jsonl 2>&1; echo ab2=$?
cat gpurun_out/tile_ab2.jsonl
timeout 900 python scripts/tile_ab.py 4 256 16 > gpurun_out/tile_ab4.jsonl 2>&1; echo ab4=$?
cat gpurun_out/tile_ab4.jsonl
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo tests=$?
tail -5 gpurun_out/gputests.log
timeout 900 python bench.py --steps 2 --warmup 1 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo bench=$?
tail -c 400 gpurun_out/bench_cfg2.err
