set -x
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -30 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke=$?
python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo bench=$?
tail -1 gpurun_out/bench.log | cut -c1-400
