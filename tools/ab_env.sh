# usage: ab_env.sh "ENV=a" "ENV=b" ... ; runs bench alternately twice with each env setting
for rep in 1 2; do for e in "$@"; do
  env $e timeout 300 python bench.py --no-cpu-baseline $BENCH_ARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', d['value'], d['e2e']['value'], d['with_importance']['value'], d['single_view_ms'], d['stages_ms']['project_bwd'], d['batch_step']['graph']['value'], d.get('train', {}).get('value'))"
done; done
