# Fresh ncu captures on the final build (each command first exits 0 without ncu)
set -u
timeout 200 python tools/one_step.py --workload c3 --serial > /dev/null 2>&1; echo "one_step c3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zgemm_dmma --launch-skip 207 -c 1 \
    -o gpurun_out/r01b_zgemm -f python tools/one_step.py --workload c3 --serial > /dev/null 2>&1; echo "ncu zgemm rc=$?"
timeout 200 python tools/one_step.py --workload c2 > /dev/null 2>&1; echo "one_step c2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bj_step --launch-skip 200 -c 1 \
    -o gpurun_out/r01b_bj -f python tools/one_step.py --workload c2 > /dev/null 2>&1; echo "ncu bj rc=$?"
ls -la gpurun_out/*.ncu-rep
