# compare final states of several kernel configs; usage: bash scripts/gpu_cfgcmp.sh "1 0 3 ..." (first = reference)
mkdir -p gpurun_out
for k in $1; do CDG_KCFG=$k timeout 300 python scripts/cfg_compare.py /tmp/u_$k.npy 12 3; done
python -c "
import numpy as np
ks='$1'.split(); ref=np.load(f'/tmp/u_{ks[0]}.npy')
for k in ks:
    u=np.load(f'/tmp/u_{k}.npy'); print('cfg', k, 'rel diff vs cfg', ks[0], np.abs(u-ref).max()/np.abs(ref).max())
"
