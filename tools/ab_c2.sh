for i in 1 2; do
for v in A B; do
  if [ $v = A ]; then export RRSVD_B200_LIB=$PWD/paper_1504_00992_b200/lib/librrsvd_b200_A.so; else unset RRSVD_B200_LIB; fi
  timeout 200 python bench.py --workload c2 --no-cpu-baseline > gpurun_out/c2_$v.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/c2_$v.json'));print('$v c2',d['value'])"
done; done
