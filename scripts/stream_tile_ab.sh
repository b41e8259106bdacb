for p in 0 1; do
echo pipe=$p
MLMCP_CLUSTER_PIPE=$p python scripts/cluster_check.py 3 64 16 2>&1 | tail -3
done
MLMCP_CLUSTER_PIPE=1 timeout 900 python -m pytest tests/test_gpu_mlmc.py tests/test_gpu_fe_parity.py -x -q -k "streaming or stream or cfg3 or coarse_failure" > gpurun_out/pt_pipe.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pt_pipe.log
MLMCP_CLUSTER_PIPE=1 python scripts/config_runs.py 3
MLMCP_CLUSTER_PIPE=0 python scripts/config_runs.py 3
