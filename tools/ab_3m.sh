for v in 1 3; do RRSVD_B200_GEMM_3M=$v timeout 300 python bench.py --no-cpu-baseline > gpurun_out/c3_3m$v.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/c3_3m$v.json'));r=d['roofline']
print('3M=$v c3',d['value'],'e2e',d['e2e']['value'],'gemm TF/s',r['achieved'],{k:v['tflops'] for k,v in r['stages'].items()})"; done
