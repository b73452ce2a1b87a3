# full GPU suite + smoke with the defaults (emulated A-products on), then the C3 bench with and without
set -u
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/full_suite.log 2>&1; echo "suite rc=$?"; tail -3 gpurun_out/full_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_def.json 2> gpurun_out/bench_def.err; echo "bench rc=$?"
RRSVD_B200_OZAKI=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_dmma.json 2> gpurun_out/bench_dmma.err
python - <<'PY'
import json
for f in ("bench_def", "bench_dmma"):
    d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
    r = d["roofline"]
    print(f, d["value"], d["e2e"]["value"], r["frac"], r.get("frac_executed"), json.dumps(r.get("emulated_a_products"))[:400])
PY
