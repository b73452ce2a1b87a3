for v in 0 1; do RRSVD_B200_BJ_PER_STEP=$v timeout 400 python tools/one_step.py --workload c3det 2>&1 | grep "ms per step" | tail -1 | sed "s/^/per_step=$v /"; done
