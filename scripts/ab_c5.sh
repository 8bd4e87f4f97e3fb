for lib in paper_2205_07824_b200/lib/libldgb200.so variants/w5/libldgb200.so; do
  LDGB200_LIB=$PWD/$lib timeout 600 python scripts/sweep_config5.py 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', [(r['p'], round(r['gdofs'],1)) for r in d['rows']])"
done
