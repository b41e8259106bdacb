#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python scripts/tile_ab.py 4 256 16 region,regionw 2>&1 | grep -E "mode|vs_first" | cut -c1-330
