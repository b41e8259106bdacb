timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
python scripts/config_runs.py 2 4
