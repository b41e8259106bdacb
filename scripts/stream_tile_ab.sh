export MLMCP_TILE_CFG=5
timeout 600 python -m pytest tests/test_gpu_mlmc.py tests/test_gpu_fe_parity.py -x -q -k "streaming or stream or cfg2 or cfg4 or ragged" > gpurun_out/pt_stream.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pt_stream.log
export MLMCP_STREAM_IMPL=4
for c in 1 5; do
 echo "tilecfg=$c"
 MLMCP_TILE_CFG=$c timeout 300 python scripts/microbench_stream.py 2 64 16 3
 MLMCP_TILE_CFG=$c timeout 300 python scripts/microbench_stream.py 4 16 8 3
 MLMCP_TILE_CFG=$c timeout 300 python scripts/microbench_stream.py 2 512 8 2
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/tile_launches_c5.csv python scripts/microbench_stream.py 2 64 4 0 > /dev/null 2>&1; echo l=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tile_persist -s 20 -c 1 -f -o gpurun_out/prof_persist python scripts/microbench_stream.py 2 64 4 0 > gpurun_out/persist_ncu.log 2>&1; echo n=$?
