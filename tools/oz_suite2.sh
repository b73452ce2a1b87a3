# full GPU suite with the defaults, then the C3 bench A/B over the tail / span switches
set -u
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/full_suite.log 2>&1; echo "suite rc=$?"; tail -3 gpurun_out/full_suite.log
for cfg in "" "RRSVD_B200_OZAKI_TAIL=2" "RRSVD_B200_OZAKI_TAIL=2 RRSVD_B200_SPAN_PASSES=1" "RRSVD_B200_OZAKI=0"; do
  env $cfg timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); r=d['roofline']; e=r['emulated_a_products']
print('cfg=[$cfg]', d['value'], d['e2e']['value'], 'qr', r['stages'].get('qr_gram'), r['stages'].get('qr_apply'), 'dmmaA', r['stages'].get('rrsvd_A_products'), 'oz', e.get('ms_per_step'), e.get('a_preparation_ms_per_step'))"
done
