python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python scripts/parareal_timeline.py 2>&1 | grep -v "0.00[0-9] ms"
MLMCP_PREDICTOR=0 python bench.py --steps 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('pred off', d['ms_per_step'], d['detail'])"
python bench.py --steps 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('pred on', d['ms_per_step'], d['detail'])"
