# Ozaki A-products: tests at the headline shape, launch list of a serial C3 step, one --set full capture of oz_gemm
set -u
export RRSVD_B200_OZAKI=16
timeout 600 python -m pytest tests/test_gpu_headline.py -x -q > gpurun_out/oz3_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/oz3_tests.log
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv \
    --log-file gpurun_out/oz3_onestep.csv python tools/one_step.py --workload c3 --serial > /dev/null 2>&1; echo "list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:oz_gemm --launch-skip 20 -c 1 \
    -o gpurun_out/oz3_gemm -f python tools/one_step.py --workload c3 --serial > /dev/null 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:oz_resid_a --launch-skip 2 -c 1 \
    -o gpurun_out/oz3_resa -f python tools/one_step.py --workload c3 --serial > /dev/null 2>&1; echo "ncu rc=$?"
