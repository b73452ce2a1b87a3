timeout 300 python bench.py --workload c2 --no-cpu-baseline --steps 3 > gpurun_out/fin3_c2.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/fin3_c2.json'));print('c2',d['value'],d['e2e']['value'])"
timeout 300 python bench.py --workload c2 --no-cpu-baseline > gpurun_out/fin3_c2_10.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/fin3_c2_10.json'));print('c2 10 steps',d['value'],d['e2e']['value'])"
timeout 1100 python tools/measure_configs.py > gpurun_out/fin3_configs.jsonl 2>/dev/null; grep full_svd gpurun_out/fin3_configs.jsonl | cut -c1-200
timeout 1300 python bench.py --workload c3det --no-cpu-baseline > gpurun_out/fin3_c3det.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/fin3_c3det.json'));print('c3det',d['value'])"
