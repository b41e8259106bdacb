#!/bin/bash
# round-2 GPU call K: band path with 8-row strips — A/B, parity, ncu, bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python scripts/tile_ab.py 2 1024 64 region,band > gpurun_out/band_ab2.jsonl 2>&1; echo ab2=$?
cut -c1-300 gpurun_out/band_ab2.jsonl
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo tests=$?
grep -E "passed|failed|FAILED" gpurun_out/gputests.log | head -20
timeout 900 ncu --set full --clock-control none --import-source on -k regex:band_propagate -c 1 -f -o gpurun_out/prof_band python scripts/tile_ab.py 2 14 16 band > gpurun_out/ncu_band.log 2>&1; echo ncu=$?
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo bench=$?
cut -c1-400 gpurun_out/bench_cfg2.json; tail -c 600 gpurun_out/bench_cfg2.err
