# A/B of the steady-state predictor on the streaming path (configs 2-4):
# default (extrapolation only) vs MLMCP_PREDICTOR=all (periodic COCG + ss guess)
for pred in 1 all; do
  echo "== MLMCP_PREDICTOR=$pred"
  MLMCP_PREDICTOR=$pred timeout 300 python scripts/microbench_stream.py 3 256 16
  MLMCP_PREDICTOR=$pred timeout 300 python scripts/microbench_stream.py 2 64 16
  MLMCP_PREDICTOR=$pred timeout 300 python scripts/microbench_stream.py 4 16 8
done
