# usage: ab_env.sh "ENV=a" "ENV=b" ... ; runs bench alternately twice with each env setting
for rep in 1 2; do for e in "$@"; do
  env $e timeout 300 python bench.py --no-cpu-baseline $BENCH_ARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', d['value'], d['single_view_ms'], {k:v for k,v in d['stages_ms'].items() if 'route' not in k and 'loss' not in k}, d['train']['value'])"
done; done
