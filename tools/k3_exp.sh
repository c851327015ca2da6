#!/bin/bash
# K3 timing experiments: each experiment build (librsr_x*.so) vs librsr.so, k3_bench cases.
# Experiment builds (CPU side, before the gpurun call), e.g. the weights-free consumer ceiling:
#   python -c "import os,sys; sys.path.insert(0,'.'); from paper_1807_07433_b200 import build as b; \
#              b.build(out=os.path.join(b.HERE,'librsr_xnow.so'), defines=['RSR_EXP_NOWCOMP'])"
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-k3x}
for i in 1 2; do
for f in paper_1807_07433_b200/librsr.so paper_1807_07433_b200/librsr_x*.so; do
  for c in "8 720 1280 64 6 0.0" "8 720 1280 64 6 0.1"; do
    RSR_LIB=$f REPS=10 timeout 300 python tools/k3_bench.py $c 2>/dev/null | grep '"lib"' >> gpurun_out/${TAG}.jsonl
  done
done
done
python -c "
import json
for l in open('gpurun_out/${TAG}.jsonl'):
    d=json.loads(l); print(d['lib'], d['nan_band'], round(d['ms'],3), round(d['frac'],3))
"
