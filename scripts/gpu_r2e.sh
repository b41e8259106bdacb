#!/bin/bash
# round-2 GPU call E: full GPU suite, default bench (config 2), launch list of
# one config-2 level, one ncu --set full capture of the region tile kernel,
# memcheck over every kernel family
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo tests=$?
tail -15 gpurun_out/gputests.log
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo bench=$?
cat gpurun_out/bench_cfg2.json; tail -c 600 gpurun_out/bench_cfg2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2_l0.csv python scripts/tile_ab.py 2 512 16 region > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_iter -s 30 -c 1 -f -o gpurun_out/prof_tile_rg python scripts/tile_ab.py 2 1024 8 region > gpurun_out/ncu_rg.log 2>&1; echo rg=$?
TOOLS=memcheck timeout 1500 bash scripts/sanitize.sh
