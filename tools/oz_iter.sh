# one iteration on the emulated A-products: unit + headline parity, C3 bench A/B, launch list of a serial step
set -u
T=${OZ_T:-15}
timeout 300 python -m pytest tests/test_gpu_ozaki.py -x -q 2>&1 | tail -1 | sed 's/^/ozaki unit: /'
RRSVD_B200_OZAKI=$T timeout 600 python -m pytest tests/test_gpu_headline.py -x -q 2>&1 | tail -1 | sed "s/^/headline T=$T: /"
for o in 0 $T; do
  RRSVD_B200_OZAKI=$o timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/oz_bench_$o.json 2> gpurun_out/oz_bench_$o.err
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/oz_bench_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        st = d["roofline"].get("stages", {})
        print(f, d["value"], d.get("e2e", {}).get("value"), st.get("rrsvd_A_products"))
    except Exception as e:
        print(f, "ERR", e)
PY
RRSVD_B200_OZAKI=$T timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv \
    --log-file gpurun_out/oz_onestep.csv python tools/one_step.py --workload c3 --serial > /dev/null 2>&1; echo "list rc=$?"
python tools/launch_table.py gpurun_out/oz_onestep.csv 16
