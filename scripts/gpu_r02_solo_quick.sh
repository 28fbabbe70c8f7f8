cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for W in config3 config4 config4 config3; do
  timeout 600 python bench.py --workload $W --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-supplementary 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$W', d['ms_per_step'])"
done
timeout 300 python scripts/ab_flags.py base=0 nochain=8192 2>&1 | tail -2
