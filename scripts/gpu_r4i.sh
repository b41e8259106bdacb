#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mlmc.py tests/test_gpu_large_parity.py tests/test_gpu_sync_protocol.py -m gpu -q -p no:cacheprovider -k "pipelined or cfg2 or band or periodic" > gpurun_out/pipe_test.log 2>&1; echo test=$?
tail -8 gpurun_out/pipe_test.log
timeout 600 python scripts/call_timeline.py 2 gpurun_out/timeline_cfg2.json 2>&1 | grep -E "band|wall|periodic"
MLMCP_PIPELINE=0 timeout 600 python scripts/call_timeline.py 2 gpurun_out/timeline_cfg2_serial.json 2>&1 | grep -E "band|wall|periodic"
