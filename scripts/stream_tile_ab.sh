timeout 900 python -m pytest tests/test_gpu_mlmc.py tests/test_gpu_fe_parity.py -x -q -k "streaming or stream or cfg2 or cfg4 or ragged or agree" > gpurun_out/pt_stream1.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pt_stream1.log
export MLMCP_STREAM_IMPL=4
timeout 300 python scripts/microbench_stream.py 2 64 64 2
timeout 300 python scripts/microbench_stream.py 4 16 32 2
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/stream_launches_v15.csv python scripts/microbench_stream.py 2 64 8 0 > /dev/null 2>&1; echo l=$?
