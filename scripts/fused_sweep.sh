# estimate time: separate launches, one fused launch, Parareal-only persistent launch on N slots
b() { timeout 300 python bench.py --steps 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'])"; }
echo -n "all-in-one "; MLMCP_FUSED=all b
for r in 32 64; do echo -n "all-in-one reserve=$r "; MLMCP_FUSED=all MLMCP_FUSED_RESERVE=$r b; done
for r in auto 64 96; do
  echo -n "split pr_ctas=$r "
  if [ "$r" = auto ]; then unset MLMCP_PR_CTAS; else export MLMCP_PR_CTAS=$r; fi
  b
done
