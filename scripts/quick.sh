# quick GPU loop: parity tests, short bench, step + field phase timings
tag=${1:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_tests.log
tail -3 gpurun_out/${tag}_tests.log
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/${tag}_bench.log 2>&1
tail -1 gpurun_out/${tag}_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value %.4g ms %.4f field %.4f parity %s e2e %.4g' % (d['value'], d['ms_per_step'], d['roofline']['launch_ms'], d.get('parity_vs_oracle'), d['e2e']['value']))"
[ -f paper_1711_08604_b200/lib/libafd_b200_timing.so ] && timeout 120 python scripts/step_timing.py 2>&1 | tail -14
[ -f paper_1711_08604_b200/lib/libafd_b200_ftiming.so ] && timeout 120 python scripts/field_timing.py c1 2>&1 | tail -6
