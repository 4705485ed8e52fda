#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2oo_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2oo_tests.log
for c in c4 c2 c0; do st=10; [ $c == c0 ] && st=30
  echo -n "$c "; timeout 900 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline 2>/dev/null | tee gpurun_out/r2oo_$c.json | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('%.4e e2e %.4e field %.4f frac %.3f parity %s split %s' % (d['value'], d['e2e']['value'], r['launch_ms'], r['frac'], d['parity_vs_oracle'], {k: r.get('split',{}).get(k) for k in ('rows_1024','rows_4096','twopass_rows')}))"; done
for a in "1048576 16384 1 1" "65536 4096 1 1"; do python scripts/probe_fast.py $a 3 | tail -1; done
