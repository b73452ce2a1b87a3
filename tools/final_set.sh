# all secondary bench lines + config measurements on the current build (outputs in gpurun_out/)
for w in c3p100 c2 c5 c4; do
  timeout 900 python bench.py --workload $w --no-cpu-baseline > gpurun_out/fin_$w.json 2> gpurun_out/fin_$w.err
  python -c "import json;d=json.load(open('gpurun_out/fin_$w.json'));e=d.get('e2e') or {};print('$w',d['value'],d['unit'],'e2e',e.get('value'))" || tail -2 gpurun_out/fin_$w.err
done
timeout 1100 python tools/measure_configs.py > gpurun_out/fin_configs.jsonl 2> gpurun_out/fin_configs.err; cut -c1-200 gpurun_out/fin_configs.jsonl
timeout 1300 python bench.py --workload c3det --no-cpu-baseline > gpurun_out/fin_c3det.json 2> gpurun_out/fin_c3det.err
python -c "import json;d=json.load(open('gpurun_out/fin_c3det.json'));print('c3det',d['value'])"
