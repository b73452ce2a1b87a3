# A/B: lanes per batched sweep on the headline workload, alternated
for T in 2 3 4 2 3 4; do RRSVD_B200_LANES=$T timeout 300 python bench.py --no-cpu-baseline > gpurun_out/lanes_$T.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/lanes_$T.json'));print('LANES=$T c3',d['value'],d['device_time_per_step_ms'])"; done
