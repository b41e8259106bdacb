timeout 900 python -m pytest tests/test_gpu_mlmc.py tests/test_gpu_fe_parity.py -x -q -k "streaming or stream or cfg2 or cfg4 or cfg3 or ragged or agree or coarse_failure" > gpurun_out/pt_stream1.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pt_stream1.log
python scripts/config_runs.py 2 4
