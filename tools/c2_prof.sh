# C2 deterministic: launch list of one step and a --set full capture of the longest block-Jacobi launch
set -u
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__cluster_size --clock-control none --csv \
    --log-file gpurun_out/c2_onestep.csv python tools/one_step.py --workload c2 --serial > /dev/null 2>&1; echo "list rc=$?"
python tools/launch_table.py gpurun_out/c2_onestep.csv 12
IDX=$(python tools/pick_launch.py gpurun_out/c2_onestep.csv bj_step); echo "bj_step skip=$IDX"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bj_step --launch-skip $IDX -c 1 \
    -o gpurun_out/c2_bj -f python tools/one_step.py --workload c2 --serial > /dev/null 2>&1; echo "ncu rc=$?"
