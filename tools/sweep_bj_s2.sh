for S in 0 1 2 4 8; do RRSVD_B200_BJ_S=$S timeout 300 python tools/jac_probe.py 1000 2000 4000 | tr '\n' ' ' | sed "s/^/S=$S /"; echo; done
