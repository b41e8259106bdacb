#!/bin/bash
# round-2 GPU call I: cluster-resident band path (256^2) — A/B vs the tile path, parity
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python scripts/tile_ab.py 2 256 32 region,band > gpurun_out/band_ab.jsonl 2>&1; echo ab=$?
cut -c1-400 gpurun_out/band_ab.jsonl; tail -5 gpurun_out/band_ab.jsonl | grep -i error
timeout 600 python scripts/tile_ab.py 2 1024 64 region,band > gpurun_out/band_ab2.jsonl 2>&1; echo ab2=$?
cut -c1-400 gpurun_out/band_ab2.jsonl
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo tests=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/gputests.log | head -20
