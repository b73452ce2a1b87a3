# jacobi kernel A/B: launch lists of a C1 decimation and a C3 step with the CTA-pair Jacobi and the cluster kernel
for J in 1 0; do
RRSVD_B200_JAC_PAIR=$J timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/jab_c1_$J.csv python tools/one_decimation.py --n 512 --k 64 --p 10 --reps 2 > /dev/null 2>&1
RRSVD_B200_JAC_PAIR=$J timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/jab_c3_$J.csv python tools/one_step.py --workload c3 > /dev/null 2>&1
RRSVD_B200_JAC_PAIR=$J RRSVD_B200_DEBUG=1 timeout 300 python tools/one_decimation.py --n 512 --k 64 --p 10 --reps 1 > gpurun_out/jab_dbg_$J.log 2>&1
done
echo done
