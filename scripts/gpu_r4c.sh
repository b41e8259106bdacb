#!/bin/bash
# ncu --set full of the recompute-w tile iteration kernel on a config-4 level-0 batch
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_iter_rw -s 30 -c 1 -f -o gpurun_out/prof_tile_rw python scripts/tile_ab.py 4 128 6 region > gpurun_out/ncu_rw.log 2>&1; echo rw=$?
tail -3 gpurun_out/ncu_rw.log | cut -c1-300
