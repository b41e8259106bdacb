set -x
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke=$?
python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo bench=$?
tail -1 gpurun_out/bench.log | cut -c1-300
ncu --set full --clock-control none --import-source on -k regex:tile_iter -s 20 -c 1 -f -o gpurun_out/prof_tile_v12 python scripts/microbench_stream.py 2 64 4 0 > gpurun_out/tile_ncu.log 2>&1; echo n=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/stream_launches_v12.csv python scripts/microbench_stream.py 2 64 4 0 > /dev/null 2>&1; echo l=$?
