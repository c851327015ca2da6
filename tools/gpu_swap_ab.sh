#!/bin/bash
# A/B of K3's swapped half loads for G = 4 (RSR_K3_SWAP=0: the unswapped loads), per-phase
# times at cP and c1, and K3 alone at the cP shape (rho = 2, 4, 5) and the c5 shape
# (D = 32 at rho = 4; D = 12 at rho = 7 and D = 64 as controls), twice alternating; then
# the whole -m gpu suite.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-swap}
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
for i in 1 2; do
  for rc in 0 1; do
    for c in "cP 8" "c1 8"; do
      if [ $rc = 0 ]; then export RSR_K3_SWAP=0; else unset RSR_K3_SWAP; fi
      timeout 300 python tools/phase_bench.py $c > gpurun_out/${TAG}_tmp.txt 2>&1
      python -c "
import json
for l in open('gpurun_out/${TAG}_tmp.txt'):
    if l.startswith('{\"config'):
        d=json.loads(l); print('rc=$rc', '$c', {k: round(v,3) for k,v in d['ms'].items()}, round(d['fps'],1), d.get('clocks'))
" | tee -a gpurun_out/${TAG}.txt
    done
  done
done
unset RSR_K3_SWAP
for i in 1 2; do
  for rc in 0 1; do
    if [ $rc = 0 ]; then export RSR_K3_SWAP=0; else unset RSR_K3_SWAP; fi
    for c in "8 609 1240 30 2 0.0" "8 609 1240 30 4 0.0" "8 609 1240 30 5 0.0" "8 720 1280 32 4 0.0" "8 720 1280 12 7 0.0" "8 720 1280 64 6 0.0"; do
      REPS=10 timeout 300 python tools/k3_bench.py $c 2>/dev/null | grep '"lib"' | sed "s/^/rc=$rc /" >> gpurun_out/${TAG}_k3.txt
    done
  done
done
unset RSR_K3_SWAP
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -3 gpurun_out/${TAG}_pytest.log
