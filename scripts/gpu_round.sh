set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke=$?
python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo bench=$?
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err; echo ref=$?
python scripts/profile_seq_cfg1.py > gpurun_out/plain5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:small_propagate -s 1 -c 1 -f -o gpurun_out/prof_seq_v5 python scripts/profile_seq_cfg1.py > gpurun_out/ncu_v5.log 2>&1; echo ncu=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_v5.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
