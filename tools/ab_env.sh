# usage: ab_env.sh "ENV=a" "ENV=b" ... ; runs bench alternately twice with each env setting
for rep in 1 2; do for e in "$@"; do
  env $e timeout 300 python bench.py --no-cpu-baseline $BENCH_ARGS 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); g=lambda *k: (lambda x: [x := (x or {}).get(i) for i in k][-1])(d)
print('$e', d['value'], g('e2e','value'), g('with_importance','value'), d['single_view_ms'],
      {k: v for k, v in d['stages_ms'].items() if 'route' not in k}, g('batch_step','graph','value'), g('train','value'))"
done; done
