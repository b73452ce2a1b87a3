# what the driver runs at round end: the GPU suite, smoke, both bench arms at N=1
set -u
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/drv_suite.log 2>&1; echo "suite rc=$?"; tail -1 gpurun_out/drv_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py --impl reference > gpurun_out/drv_ref.json 2> gpurun_out/drv_ref.err; echo "ref rc=$?"
timeout 900 python bench.py > gpurun_out/drv_ours.json 2> gpurun_out/drv_ours.err; echo "ours rc=$?"
python - <<'PY'
import json
for f in ("drv_ref", "drv_ours"):
    d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
    print(f, d.get("impl"), d["value"], d["unit"], d.get("e2e", {}).get("value"), d.get("steps"), d.get("ms_per_step"), d.get("config", {}).get("workload"))
PY
