#!/bin/bash
# L2-residency probe: tile path on config-4 level-0 batches of 4..256 tasks
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for S in 4 8 12 16 32 256; do
  timeout 300 python scripts/tile_ab.py 4 $S 16 region 2>&1 | grep '"mode"' | tee -a gpurun_out/l2_probe.jsonl | cut -c1-700
done
