#!/bin/bash
# band kernel A/B iteration: call time at config-2 level-0 size, ncu of the small launch
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python scripts/tile_ab.py 2 1024 64 band > gpurun_out/band_ab.jsonl 2>&1; echo ab=$?
cut -c1-250 gpurun_out/band_ab.jsonl
timeout 900 ncu --set full --clock-control none --import-source on -k regex:band_propagate -c 1 -f -o gpurun_out/prof_band python scripts/tile_ab.py 2 14 16 band > gpurun_out/ncu_band.log 2>&1; echo ncu=$?
timeout 300 python -m pytest tests/test_gpu_large_parity.py -q -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo tests=$?; tail -1 gpurun_out/gputests.log
