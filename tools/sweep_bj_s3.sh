for S in 2 3 4 5 6; do RRSVD_B200_BJ_S=$S timeout 100 python tools/jac_probe.py 1000 2000 | tr '\n' ' ' | sed "s/^/S=$S /"; echo; done
for S in 2 3 4; do RRSVD_B200_BJ_S=$S timeout 200 python tools/jac_probe.py 4000 | sed "s/^/S=$S /"; done
