#!/bin/bash
# A/B of the attend kernels.  usage: <tag> [workload] [tokens]
set -u
TAG=${1:-ab}; W=${2:-c3_nuq3}; T=${3:-0}
OUT=gpurun_out/$TAG
mkdir -p $OUT
KVQ_WA_WH=2 timeout 300 python scripts/att_ab.py $W $T $OUT/o_new.npy 2>&1 | tail -1 | sed "s/default/WH2/" | cut -c1-60

KVQ_ATT_LEGACY=1 timeout 300 python scripts/att_ab.py $W $T $OUT/o_old.npy 2>&1 | tail -1 | cut -c1-60
python -c "
import numpy as np
b=np.load('$OUT/o_old.npy')
for f in ['o_new']:
    a=np.load('$OUT/'+f+'.npy'); r=np.abs(a-b).max(-1)/np.abs(b).max(-1); print(f, 'max rel diff vs legacy', r.max(), 'nan', np.isnan(a).sum())"
