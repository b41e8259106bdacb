#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python scripts/call_timeline.py 2 gpurun_out/timeline_cfg2.json 2>&1 | tail -40
