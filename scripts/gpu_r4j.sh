#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
MLMCP_BAND_PROF=1 timeout 300 python scripts/tile_ab.py 2 14 256 band 2>&1 | grep -E "band prof|mode" | tail -2 | cut -c1-300
timeout 300 python scripts/tile_ab.py 2 1024 256 band 2>&1 | grep -E "mode" | tail -1 | cut -c1-300
timeout 900 python -m pytest tests/test_gpu_mlmc.py tests/test_gpu_large_parity.py tests/test_gpu_sync_protocol.py -m gpu -q -p no:cacheprovider -k "pipelined or cfg2 or band" 2>&1 | tail -3
