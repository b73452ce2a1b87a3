set -u
timeout 900 python -m pytest tests/test_gpu_reference_suite.py tests/test_gpu_parity.py -m gpu -q > gpurun_out/c2p_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/c2p_tests.log
timeout 300 python tools/one_step.py --workload c2 > gpurun_out/c2p_step.log 2>&1; echo "c2 step rc=$?"; cat gpurun_out/c2p_step.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2p_launches.csv python tools/one_step.py --workload c2 > /dev/null 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/c2p_launches.csv > gpurun_out/c2p_summary.txt 2>&1; head -30 gpurun_out/c2p_summary.txt
