#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_reference_integration.py -q -p no:cacheprovider > gpurun_out/integ.log 2>&1; echo integ=$?; tail -3 gpurun_out/integ.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2_l0.csv python scripts/tile_ab.py 2 512 16 region > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_iter_rg -s 30 -c 1 -f -o gpurun_out/prof_tile_rg python scripts/tile_ab.py 2 1024 8 region > gpurun_out/ncu_rg.log 2>&1; echo rg=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_iter_kernel -s 30 -c 1 -f -o gpurun_out/prof_tile_st python scripts/tile_ab.py 2 1024 8 stored > gpurun_out/ncu_st.log 2>&1; echo st=$?
