for impl in 1 2; do
  echo "== MLMCP_STREAM_IMPL=$impl (1 two-launch, 2 cooperative)"
  MLMCP_STREAM_IMPL=$impl timeout 300 python scripts/microbench_stream.py 3 16 16
  MLMCP_STREAM_IMPL=$impl timeout 300 python scripts/microbench_stream.py 2 4 16
  MLMCP_STREAM_IMPL=$impl timeout 300 python scripts/microbench_stream.py 4 1 8
done
