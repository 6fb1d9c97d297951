# A/B of the scoring sweep (full bench lines): base12 = a variant library built by tools/variants.sh, cur = libbgs.so
for rep in 1 2; do for v in base12 cur; do
  if [ "$v" = "cur" ]; then L=libbgs.so; else L=libbgs_$v.so; fi
  BGS_LIB=$L timeout 600 python bench.py --no-cpu-baseline --steps 20 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['scoring']['value'], d['scoring']['in_flight']['value'], d['with_importance']['value'])"
done; done
