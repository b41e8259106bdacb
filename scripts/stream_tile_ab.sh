for l in 0 1 0 1; do
  MLMCP_LSGUESS=$l timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-streaming --no-e2e > gpurun_out/bench_ls$l.log 2>/dev/null
  echo ls=$l; tail -1 gpurun_out/bench_ls$l.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['detail'], d['config']['parareal_k'])"
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
python scripts/defect_parity.py 2>&1 | tail -4
