timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
RRSVD_B200_BJ_S=1 timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for v in 0 1; do RRSVD_B200_BJ_PER_STEP=$v timeout 200 python bench.py --workload c2 --no-cpu-baseline > gpurun_out/c2_ps$v.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/c2_ps$v.json'));print('per_step=$v c2',d['value'])"; done
for v in 0 1; do RRSVD_B200_BJ_S=1 RRSVD_B200_BJ_PER_STEP=$v python tools/jac_probe.py 2000 | sed "s/^/S=1 per_step=$v /"; done
python tools/jac_probe.py 2000
