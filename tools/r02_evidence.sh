# Round-2 evidence on the GPU box (each ncu command only after the same command exited 0 without it)
set -u
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "short bench rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "launch list rc=$?"
timeout 200 python tools/one_step.py --workload c3 --serial > /dev/null 2>&1; echo "one_step rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_onestep_launches.csv \
    python tools/one_step.py --workload c3 --serial > /dev/null 2>&1; echo "one_step list rc=$?"
IDX=$(python tools/pick_launch.py gpurun_out/r02_onestep_launches.csv zgemm_tma); echo "zgemm_tma skip=$IDX"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zgemm_tma --launch-skip $IDX -c 1 \
    -o gpurun_out/r02_zgemm_tma -f python tools/one_step.py --workload c3 --serial > /dev/null 2>&1; echo "ncu zgemm rc=$?"
IDX=$(python tools/pick_launch.py gpurun_out/r02_onestep_launches.csv jacobi_kernel); echo "jacobi skip=$IDX"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jacobi_kernel --launch-skip $IDX -c 1 \
    -o gpurun_out/r02_jacobi -f python tools/one_step.py --workload c3 --serial > /dev/null 2>&1; echo "ncu jacobi rc=$?"
