#!/bin/bash
# round-2 GPU call H: recompute-w region kernel (64 B/point) — A/B, parity, bench, breakdown, ncu
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python scripts/tile_ab.py 2 1024 32 regionw,region,region@2 > gpurun_out/tile_ab2.jsonl 2>&1; echo ab2=$?
cut -c1-420 gpurun_out/tile_ab2.jsonl
timeout 600 python scripts/tile_ab.py 4 256 16 regionw,region > gpurun_out/tile_ab4.jsonl 2>&1; echo ab4=$?
cut -c1-420 gpurun_out/tile_ab4.jsonl
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo tests=$?
tail -3 gpurun_out/gputests.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_iter -s 30 -c 1 -f -o gpurun_out/prof_tile_rw python scripts/tile_ab.py 2 1024 8 region > gpurun_out/ncu_rw.log 2>&1; echo ncu=$?
timeout 900 python scripts/kernel_breakdown.py 2 gpurun_out/breakdown_cfg2.json > gpurun_out/breakdown_cfg2.log 2>&1; echo bd2=$?
grep -v Warn gpurun_out/breakdown_cfg2.log | tail -16
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo bench=$?
cut -c1-300 gpurun_out/bench_cfg2.json; tail -c 600 gpurun_out/bench_cfg2.err
