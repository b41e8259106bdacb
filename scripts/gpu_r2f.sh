#!/bin/bash
# round-2 GPU call F: per-class stencil tables in the region tile kernels —
# A/B against the stored operator, parity suite, bench, ncu of the new kernel
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python scripts/tile_ab.py 2 1024 32 stored,region,region@2 > gpurun_out/tile_ab2.jsonl 2>&1; echo ab2=$?
cat gpurun_out/tile_ab2.jsonl | cut -c1-400
timeout 600 python scripts/tile_ab.py 4 256 16 stored,region > gpurun_out/tile_ab4.jsonl 2>&1; echo ab4=$?
cat gpurun_out/tile_ab4.jsonl | cut -c1-400
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo tests=$?
tail -3 gpurun_out/gputests.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_iter -s 30 -c 1 -f -o gpurun_out/prof_tile_cls python scripts/tile_ab.py 2 1024 8 region > gpurun_out/ncu_cls.log 2>&1; echo ncu=$?
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo bench=$?
cut -c1-1500 gpurun_out/bench_cfg2.json; tail -c 600 gpurun_out/bench_cfg2.err
