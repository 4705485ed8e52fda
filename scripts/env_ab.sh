# A/B over environment settings: each arg is "VAR=value" (or "-" for none), c1 bench twice each
for spec in "$@"; do
  for rep in 1 2; do
    echo -n "== $spec: "
    if [ "$spec" = "-" ]; then envs=""; else envs="$spec"; fi
    env $envs timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-parity 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value %.4g ms %.4f field %.4f e2e %.4g' % (d['value'], d['ms_per_step'], d['roofline']['launch_ms'], d['e2e']['value']))"
  done
done
