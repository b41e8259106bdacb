#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/tile_ab.py 2 1024 32 > gpurun_out/tile_ab2.jsonl 2>&1; echo ab2=$?
cat gpurun_out/tile_ab2.jsonl
timeout 600 python -m pytest tests/test_gpu_fe_parity.py tests/test_gpu_large_parity.py tests/test_gpu_reference_integration.py tests/test_gpu_mlmc.py -q -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo tests=$?
tail -5 gpurun_out/gputests.log
