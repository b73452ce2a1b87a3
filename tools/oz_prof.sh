# launch list of a serial C3 step with the emulated A-products + one --set full capture of a 48-bond oz_gemm
set -u
export RRSVD_B200_OZAKI=${OZ_T:-14}
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv \
    --log-file gpurun_out/oz_onestep.csv python tools/one_step.py --workload c3 --serial > /dev/null 2>&1; echo "list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:oz_gemm --launch-skip 12 -c 1 \
    -o gpurun_out/oz_gemm -f python tools/one_step.py --workload c3 --serial > /dev/null 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:oz_resid_a --launch-skip 0 -c 1 \
    -o gpurun_out/oz_resa -f python tools/one_step.py --workload c3 --serial > /dev/null 2>&1; echo "ncu rc=$?"
