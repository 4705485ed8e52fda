# A/B: production lib vs alternatives given as args (lib paths), c1 bench each
for lib in paper_1711_08604_b200/lib/libafd_b200.so "$@"; do
  echo "== $lib"
  AFD_LIB_PATH=$lib timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value %.4g ms %.4f field %.4f parity %s e2e %.4g' % (d['value'], d['ms_per_step'], d['roofline']['launch_ms'], d.get('parity_vs_oracle'), d['e2e']['value']))"
done
