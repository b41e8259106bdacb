python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke=$?
python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo bench=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_v15.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-streaming > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 1 -c 1 -f -o gpurun_out/prof_fused_v15 python scripts/profile_fused_cfg1.py > gpurun_out/fused_ncu.log 2>&1; echo n=$?
python scripts/config_runs.py 0 1 > gpurun_out/configs01.jsonl; echo cr=$?
