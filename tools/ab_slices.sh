timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
timeout 300 python tools/jac_probe.py 256 1000 2000 4000 | tr '\n' ' '; echo
for S in 4 7; do RRSVD_B200_BJ_S=$S timeout 100 python tools/jac_probe.py 2000 | sed "s/^/forced S=$S /"; done
timeout 300 python bench.py --workload c2 --no-cpu-baseline --steps 3 > gpurun_out/c2sl.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/c2sl.json'));print('c2',d['value'])"
timeout 300 python bench.py --workload c3p100 --no-cpu-baseline --steps 3 > gpurun_out/p100sl.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/p100sl.json'));print('c3p100',d['value'])"
