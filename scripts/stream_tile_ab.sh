python -m pytest tests/test_gpu_mlmc.py tests/test_gpu_fe_parity.py -x -q -k "streaming or stream or cfg2 or cfg4" > gpurun_out/pt_stream.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pt_stream.log
export MLMCP_STREAM_IMPL=4
for c in 1 3; do
 echo "tilecfg=$c"
 MLMCP_TILE_CFG=$c python scripts/microbench_stream.py 2 64 16 3
 MLMCP_TILE_CFG=$c python scripts/microbench_stream.py 4 16 8 3
done
MLMCP_STREAM_GRAPH=1 python scripts/microbench_stream.py 2 64 16 3
python scripts/microbench_stream.py 2 512 4 2
python scripts/microbench_stream.py 4 128 4 2
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/tile_launches_c1.csv python scripts/microbench_stream.py 2 64 4 0 > /dev/null 2>&1; echo l=$?
