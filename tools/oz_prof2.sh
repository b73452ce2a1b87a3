# --set full captures of the first (48-bond) launch of each emulation kernel in a serial C3 step
set -u
export RRSVD_B200_OZAKI=${OZ_T:-14}
for k in oz_maxexp oz_resid_a oz_resid_b oz_crt oz_gemm; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 \
      -o gpurun_out/prof_$k -f python tools/one_step.py --workload c3 --serial > /dev/null 2>&1; echo "$k rc=$?"
done
