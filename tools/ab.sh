# usage: ab.sh variantA variantB ... ; runs bench alternately twice (cur = libbgs.so, X = libbgs_X.so)
for rep in 1 2; do for v in "$@"; do
  if [ "$v" = "cur" ]; then L=libbgs.so; else L=libbgs_$v.so; fi
  BGS_LIB=$L timeout 300 python bench.py --no-cpu-baseline $BENCH_ARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d.get('train', {}); print('$v', d['value'], d['single_view_ms'], {k:v for k,v in d['stages_ms'].items() if 'route' not in k and 'loss' not in k}, 'train', t.get('value'), t.get('stages_ms', {}).get('loss'), t.get('e2e', {}).get('value'))"
done; done
