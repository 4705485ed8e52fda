# A/B: c1 bench (twice) for each lib path given (default: the production lib)
for spec in "${@:-paper_1711_08604_b200/lib/libafd_b200.so}"; do
  lib=$spec
  for rep in 1 2; do
  echo -n "== $spec: "
  AFD_LIB_PATH=$lib timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-parity 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value %.4g ms %.4f field %.4f e2e %.4g' % (d['value'], d['ms_per_step'], d['roofline']['launch_ms'], d['e2e']['value']))"
  done
done
