# every bench workload with the defaults and with RRSVD_B200_OZAKI=0
set -u
for w in c2rr c2 c3p100 c3det c4mpdo c5; do
  for o in def 0; do
    if [ $o = def ]; then e=""; else e="RRSVD_B200_OZAKI=0"; fi
    env $e timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/w.json 2>/dev/null
    python -c "
import json
try:
    d=json.loads(open('gpurun_out/w.json').read().strip().splitlines()[-1]); print('$w', '$o', d['value'], d['unit'], d.get('e2e',{}).get('value'))
except Exception as ex: print('$w', '$o', 'ERR', ex)"
  done
done
