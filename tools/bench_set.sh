# quick bench set (device values only): bash tools/bench_set.sh c2 c3 ...
for w in "$@"; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bs_$w.json 2>gpurun_out/bs_$w.err
  python -c "import json;d=json.load(open('gpurun_out/bs_$w.json'));print('$w',d['value'],d['unit'],'e2e',d['e2e']['value'])" || tail -3 gpurun_out/bs_$w.err
done
