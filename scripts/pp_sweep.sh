for m in 0 1 2; do
  echo "== mode $m" 
  AFD_FIELD_PP=$m timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['launch_ms'], d.get('parity_vs_oracle'), d['e2e']['value'])"
  AFD_FIELD_PP=$m timeout 300 python scripts/field_timing.py c1 2>&1 | tail -6
done
