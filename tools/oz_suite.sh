# The whole GPU suite with the emulated A-products (RRSVD_B200_OZAKI=${OZ_T:-14}), then the C3 bench A/B
set -u
T=${OZ_T:-14}
RRSVD_B200_OZAKI=$T timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/oz_suite.log 2>&1; echo "suite (T=$T) rc=$?"; tail -3 gpurun_out/oz_suite.log
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
