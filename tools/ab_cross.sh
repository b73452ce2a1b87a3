timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for v in 0 1; do RRSVD_B200_BJ_CROSS=$v RRSVD_B200_DEBUG=1 timeout 300 python tools/jac_probe.py 256 1000 2000 2>&1 | grep "svd_full\|block jacobi [0-9]" | tr '\n' ' ' | sed "s/^/cross=$v /"; echo; done
for v in 0 1; do RRSVD_B200_BJ_CROSS=$v timeout 300 python bench.py --workload c2 --no-cpu-baseline --steps 3 > gpurun_out/c2x$v.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/c2x$v.json'));print('cross=$v c2',d['value'])"; done
