#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:band_propagate -c 1 -f -o gpurun_out/prof_band python scripts/tile_ab.py 2 14 16 band > gpurun_out/ncu_band.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_band.log
