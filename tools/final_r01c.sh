set -u
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fc_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/fc_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/fc_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/fc_tests.log
timeout 900 python bench.py > gpurun_out/fc_bench.json 2> gpurun_out/fc_bench.err; echo "bench rc=$?"; head -c 250 gpurun_out/fc_bench.json; echo
