b() { timeout 300 python bench.py --steps 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['detail']['pcg_iterations_sequential'])"; }
for r in 1e-8 1e-9 1e-10 1e-11 1e-12; do echo -n "ss_rtol=$r "; MLMCP_SS_RTOL=$r b; done
