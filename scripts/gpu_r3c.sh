#!/bin/bash
# band-path guess batching (8 rows) + source profile from the class table:
# band tests, phase cycles, level-0 A/B, the config-2 bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "band or large or sync or cfg2" > gpurun_out/gputests_band.log 2>&1; echo tests=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/gputests_band.log | head -20
MLMCP_BAND_PROF=1 timeout 300 python scripts/tile_ab.py 2 14 64 band 2>&1 | tail -4
timeout 300 python scripts/tile_ab.py 2 1024 256 band 2>&1 | tail -2
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err; echo bench=$?
python -c "import json; d=json.load(open('gpurun_out/bench_c.json')); print(d['ms_per_step'], d['value'], d['e2e']['value'], d['detail'])"
