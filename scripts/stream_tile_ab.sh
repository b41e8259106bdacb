timeout 600 python -m pytest tests/test_gpu_mlmc.py tests/test_gpu_fe_parity.py -x -q -k "streaming or stream or cfg2 or cfg4 or ragged or agree" > gpurun_out/pt_stream.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pt_stream.log
export MLMCP_STREAM_IMPL=4
for pdl in 0 1 0 1; do
echo pdl=$pdl
MLMCP_TILE_PDL=$pdl timeout 300 python scripts/microbench_stream.py 2 64 16 3
MLMCP_TILE_PDL=$pdl timeout 300 python scripts/microbench_stream.py 2 512 8 2
MLMCP_TILE_PDL=$pdl timeout 300 python scripts/microbench_stream.py 4 128 4 2
done
