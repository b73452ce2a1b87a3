timeout 700 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for L in 2 3 4; do RRSVD_B200_LANES=$L timeout 300 python bench.py --no-cpu-baseline > gpurun_out/c3_l$L.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/c3_l$L.json'));print('lanes=$L c3',d['value'],d['e2e']['value'])"; done
timeout 200 python bench.py --workload c2 --no-cpu-baseline > gpurun_out/c2_cp.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/c2_cp.json'));print('c2',d['value'])"
