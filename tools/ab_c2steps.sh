for S in 3 10; do timeout 300 python bench.py --workload c2 --no-cpu-baseline --steps $S > gpurun_out/c2_s$S.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/c2_s$S.json'));print('steps=$S c2',d['value'])"; done
RRSVD_B200_DEBUG=1 timeout 200 python tools/one_step.py --workload c2 2>&1 | grep "block jacobi [0-9]" | sort | uniq -c
