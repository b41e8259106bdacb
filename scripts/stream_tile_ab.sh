MLMCP_TILE_CFG=5 timeout 600 python -m pytest tests/test_gpu_mlmc.py -x -q -k "ragged" > gpurun_out/pt_stream.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pt_stream.log
export MLMCP_STREAM_IMPL=4
for c in 1 5 3; do
echo cfg=$c
MLMCP_TILE_CFG=$c timeout 300 python scripts/microbench_stream.py 2 64 16 3
MLMCP_TILE_CFG=$c timeout 300 python scripts/microbench_stream.py 2 512 8 2
done
