#!/bin/bash
# Re-entry check of HEAD: full GPU suite, smoke, config-2 bench, all configs
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
set -x
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo bench=$?
tail -1 gpurun_out/bench.log | cut -c1-400
timeout 900 python scripts/config_runs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo configs=$?
cut -c1-300 gpurun_out/configs.jsonl
