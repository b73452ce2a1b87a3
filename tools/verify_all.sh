set -u
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/va_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/va_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/va_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/va_tests.log
