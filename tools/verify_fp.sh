set -u
timeout 600 python tools/fp_probe.py > gpurun_out/fp_probe2.log 2>&1; echo "probe rc=$?"; grep -c MISMATCH gpurun_out/fp_probe2.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/vf_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/vf_tests.log
