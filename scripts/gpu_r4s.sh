#!/bin/bash
# final captures: ncu --set full of the band kernel, launch list of the bench command
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:band_propagate -c 1 -f -o gpurun_out/prof_band python scripts/tile_ab.py 2 14 16 band > gpurun_out/ncu_band.log 2>&1; echo ncu=$?
ITS=$(grep '"mode"' gpurun_out/ncu_band.log | tail -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['pcg_iterations'])")
python scripts/ncu_summary.py gpurun_out/prof_band.ncu-rep band_propagate_kernel $ITS 65025 452929 0 gpurun_out/r2_v10_ncu_band.json "config-2 level-0 batch, 14 tasks x 16 steps (2 per cluster, 7 clusters; scripts/tile_ab.py 2 14 16 band)" > gpurun_out/ncu_summary.log 2>&1; echo summary=$?
cp profiles/ncu_top_kernel.json gpurun_out/ncu_top_kernel.json
python scripts/ncu_lines.py gpurun_out/prof_band.ncu-rep 40 > gpurun_out/r2_v10_ncu_band_lines.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_v10_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launches.log 2>&1; echo launches=$?
wc -l gpurun_out/r2_v10_launches.csv
