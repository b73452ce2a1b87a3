# Final round evidence (run on the GPU box; each ncu command only after the same command exited 0 without it)
set -u
timeout 900 python bench.py > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "short bench rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "launch list rc=$?"
timeout 200 python tools/one_step.py --workload c3 --serial > /dev/null 2>&1; echo "one_step rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zgemm_dmma --launch-skip 207 -c 1 \
    -o gpurun_out/ev_zgemm -f python tools/one_step.py --workload c3 --serial > /dev/null 2>&1; echo "ncu zgemm rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chol_inv --launch-skip 40 -c 1 \
    -o gpurun_out/ev_chol -f python tools/one_step.py --workload c3 --serial > /dev/null 2>&1; echo "ncu chol rc=$?"
timeout 200 python tools/one_step.py --workload c2 > /dev/null 2>&1; echo "one_step c2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bj_sweep --launch-skip 10 -c 1 \
    -o gpurun_out/ev_bj -f python tools/one_step.py --workload c2 > /dev/null 2>&1; echo "ncu bj rc=$?"
