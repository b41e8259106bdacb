for l in 0 1; do
  echo ls=$l
  MLMCP_LSGUESS=$l MLMCP_STREAM_IMPL=4 timeout 300 python scripts/microbench_stream.py 2 64 128 2
done
timeout 900 python -m pytest tests/test_gpu_mlmc.py tests/test_gpu_fe_parity.py -x -q -k "streaming or stream or cfg2 or cfg4 or ragged or agree" > gpurun_out/pt_stream1.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pt_stream1.log
python scripts/config_runs.py 2
