export MLMCP_STREAM_IMPL=4
ncu --set full --clock-control none --import-source on -k regex:tile_iter -s 20 -c 1 -f -o gpurun_out/prof_tile_v12b python scripts/microbench_stream.py 2 64 4 0 > gpurun_out/tile_ncu.log 2>&1; echo n=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/stream_launches_v12b.csv python scripts/microbench_stream.py 2 64 4 0 > /dev/null 2>&1; echo l=$?
