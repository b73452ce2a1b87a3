# Round-2 final evidence: default bench line (with the CPU baseline leg), the all-DMMA A/B line,
# the launch list of a serial C3 step, and --set full captures of the dominant kernels of that step
# (each ncu command only after the same command exited 0 without ncu)
set -u
timeout 900 python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err; echo "bench rc=$?"
RRSVD_B200_OZAKI=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/fin_bench_dmma.json 2> /dev/null; echo "bench dmma rc=$?"
timeout 300 python tools/one_step.py --workload c3 --serial > /dev/null 2>&1; echo "one_step rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv \
    --log-file gpurun_out/fin_onestep.csv python tools/one_step.py --workload c3 --serial > /dev/null 2>&1; echo "list rc=$?"
for k in oz_gemm_persistent oz_resid_a oz_crt oz_resid_b chol_inv; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 \
      -o gpurun_out/fin_$k -f python tools/one_step.py --workload c3 --serial > /dev/null 2>&1; echo "$k rc=$?"
  ncu -i gpurun_out/fin_$k.ncu-rep --page raw --csv > gpurun_out/fin_${k}_raw.csv 2>/dev/null
done
IDX=$(python tools/pick_launch.py gpurun_out/fin_onestep.csv zgemm_tma); echo "zgemm_tma skip=$IDX"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zgemm_tma --launch-skip $IDX -c 1 \
    -o gpurun_out/fin_zgemm_tma -f python tools/one_step.py --workload c3 --serial > /dev/null 2>&1; echo "ncu zgemm rc=$?"
ncu -i gpurun_out/fin_zgemm_tma.ncu-rep --page raw --csv > gpurun_out/fin_zgemm_tma_raw.csv 2>/dev/null
cuobjdump -sass paper_1504_00992_b200/lib/librrsvd_b200.so 2>/dev/null | grep -o "UTCIMMA[A-Z0-9_.]*\|UTMALDG[A-Z0-9_.]*\|UTCBAR[A-Z0-9_.]*\|UTCATOMSWS[A-Z0-9_.]*\|LDTM[A-Z0-9_.]*\|DMMA[A-Z0-9_.]*" | sort | uniq -c > gpurun_out/fin_sass_grep.txt
