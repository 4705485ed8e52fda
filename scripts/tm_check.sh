timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in 1 0; do
  echo -n "AFD_FIELD_TMEM=$v: "
  AFD_FIELD_TMEM=$v timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value %.4g ms %.4f field %.4f parity %s e2e %.4g' % (d['value'], d['ms_per_step'], d['roofline']['launch_ms'], d.get('parity_vs_oracle'), d['e2e']['value']))"
done
