# Emulated A-products (RRSVD_B200_OZAKI = moduli): parity suites and the C3 bench, A/B against the DMMA zgemm
set -u
T=${OZ_T:-16}
timeout 300 python -m pytest tests/test_gpu_ozaki.py -x -q > gpurun_out/oz_tests0.log 2>&1; echo "ozaki tests rc=$?"; tail -2 gpurun_out/oz_tests0.log
RRSVD_B200_OZAKI=$T timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_parity.py -x -q > gpurun_out/oz_tests.log 2>&1; echo "parity (T=$T) rc=$?"; tail -3 gpurun_out/oz_tests.log
for o in 0 $T ${OZ_T2:-}; do
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
