b() { timeout 300 python bench.py --steps 8 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['detail']['pcg_iterations_sequential'], d['detail']['pcg_iterations_parareal_fine'], d['detail']['pcg_iterations_parareal_coarse'])"; }
for o in 1 2 3; do echo -n "order=$o "; MLMCP_ORDER=$o b; done
