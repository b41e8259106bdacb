#!/bin/bash
# band path: one launch per call (mixed dt), low-priority band stream, two calls in flight
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_mlmc.py tests/test_gpu_large_parity.py tests/test_gpu_sync_protocol.py -m gpu -q -p no:cacheprovider -k "pipelined or cfg2 or band" > gpurun_out/pipe_test.log 2>&1; echo test=$?
tail -5 gpurun_out/pipe_test.log
timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_pipe.log 2> gpurun_out/bench_pipe.err; echo bench_pipe=$?
tail -1 gpurun_out/bench_pipe.log | cut -c1-300
tail -3 gpurun_out/bench_pipe.err
MLMCP_PIPELINE=0 timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_serial.log 2> gpurun_out/bench_serial.err; echo bench_serial=$?
tail -1 gpurun_out/bench_serial.log | cut -c1-300
