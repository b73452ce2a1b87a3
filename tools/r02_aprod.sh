# ncu capture of the dominant RRSVD A-product launch (48-bond Y = A Q batch, grid 3072) of a serial C3 step
set -u
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv \
    --log-file gpurun_out/r02_onestep_grid.csv python tools/one_step.py --workload c3 --serial > /dev/null 2>&1
IDX=$(python tools/pick_launch.py gpurun_out/r02_onestep_grid.csv zgemm_tma 3072); echo "aprod skip=$IDX"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zgemm_tma --launch-skip $IDX -c 1 \
    -o gpurun_out/r02_zgemm_aprod -f python tools/one_step.py --workload c3 --serial > /dev/null 2>&1; echo "ncu rc=$?"
RRSVD_B200_GEMM_TMA=0 timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv \
    --log-file gpurun_out/r02_onestep_grid_notma.csv python tools/one_step.py --workload c3 --serial > /dev/null 2>&1
IDX=$(python tools/pick_launch.py gpurun_out/r02_onestep_grid_notma.csv zgemm_dmma 3072); echo "aprod (cp.async) skip=$IDX"
RRSVD_B200_GEMM_TMA=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:zgemm_dmma --launch-skip $IDX -c 1 \
    -o gpurun_out/r02_zgemm_aprod_cpasync -f python tools/one_step.py --workload c3 --serial > /dev/null 2>&1; echo "ncu rc=$?"
