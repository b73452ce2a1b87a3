timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
timeout 300 python tools/jac_probe.py 256 1000 2000 4000 | tr '\n' ' '; echo
timeout 300 python bench.py --workload c2 --no-cpu-baseline --steps 3 > gpurun_out/c2id.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/c2id.json'));print('c2',d['value'])"
