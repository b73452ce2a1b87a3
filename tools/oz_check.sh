# headline parity + variants + C3 / C2rr benches with the current defaults
set -u
timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_variants.py -q -x 2>&1 | tail -2
for w in c3 c2rr c3p100; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['e2e']['value'])"
done
