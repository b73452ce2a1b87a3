timeout 700 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
RRSVD_B200_DEBUG=1 timeout 200 python tools/one_step.py --workload c3 2>&1 | grep "jacobi 1" | awk '{print $2, $NF, $(NF-1)}' | sort | uniq -c | sort -rn | head -5
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/c3_j.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/c3_j.json'));print('c3',d['value'],d['e2e']['value'])"
for v in 0 1; do RRSVD_B200_GEMM_3M64=$v timeout 200 python bench.py --workload c2 --no-cpu-baseline > gpurun_out/c2_m$v.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/c2_m$v.json'));print('3M64=$v c2',d['value'])"; done
