for S in 0 2 4; do RRSVD_B200_BJ_S=$S timeout 200 python bench.py --workload c2 --no-cpu-baseline > gpurun_out/c2_s$S.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/c2_s$S.json'));print('S=$S c2',d['value'])"; done
for S in 0 2 8; do RRSVD_B200_BJ_S=$S python tools/jac_probe.py 2000 | sed "s/^/S=$S /"; done
