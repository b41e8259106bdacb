for o in 4 7; do
echo order=$o
MLMCP_CLUSTER_ORDER=$o python scripts/cluster_check.py 3 64 64 2>&1 | tail -3
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
python scripts/config_runs.py 3 2 4
