timeout 600 python -m pytest tests/test_gpu_mlmc.py tests/test_gpu_fe_parity.py -x -q -k "streaming or stream or cfg2 or cfg4 or ragged or agree" > gpurun_out/pt_stream1.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pt_stream1.log
export MLMCP_STREAM_IMPL=4
for r in 1 2; do
timeout 300 python scripts/microbench_stream.py 2 64 16 3
timeout 300 python scripts/microbench_stream.py 2 512 8 2
timeout 300 python scripts/microbench_stream.py 4 128 4 2
done
