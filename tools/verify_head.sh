# Re-verify the current HEAD on a B200: smoke, the full GPU suite, the headline bench.
set -u
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/vh_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/vh_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/vh_tests.log
timeout 900 python bench.py > gpurun_out/vh_bench.json 2> gpurun_out/vh_bench.err; echo "bench rc=$?"; cat gpurun_out/vh_bench.json | head -c 600
