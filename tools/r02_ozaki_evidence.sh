# Round-2 evidence for the emulated A-products: bench line (defaults), launch list of a serial C3
# step, --set full captures of the INT8 GEMM and the A-residue kernel (first 48-bond launches)
set -u
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv \
    --log-file gpurun_out/ev_onestep.csv python tools/one_step.py --workload c3 --serial > /dev/null 2>&1; echo "list rc=$?"
for k in oz_gemm_persistent oz_resid_a; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 \
      -o gpurun_out/ev_$k -f python tools/one_step.py --workload c3 --serial > /dev/null 2>&1; echo "$k rc=$?"
  ncu -i gpurun_out/ev_$k.ncu-rep --page raw --csv > gpurun_out/ev_${k}_raw.csv 2>/dev/null
  ncu -i gpurun_out/ev_$k.ncu-rep --page details --csv > gpurun_out/ev_${k}_details.csv 2>/dev/null
done
cuobjdump -sass paper_1504_00992_b200/lib/librrsvd_b200.so 2>/dev/null | grep -o "UTCIMMA[A-Z0-9_.]*\|UTMALDG[A-Z0-9_.]*\|UTCBAR[A-Z0-9_.]*\|UTCATOMSWS[A-Z0-9_.]*\|LDTM[A-Z0-9_.]*" | sort | uniq -c > gpurun_out/ev_sass_tcgen05.txt
