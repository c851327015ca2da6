#!/bin/bash
# Per-phase A/B (tools/phase_bench.py c5 8) of librsr.so and every librsr_x*.so, twice
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-pab}
for i in 1 2; do
for f in paper_1807_07433_b200/librsr.so paper_1807_07433_b200/librsr_x*.so; do
  RSR_LIB=$f timeout 300 python tools/phase_bench.py ${CFG:-c5 8} > gpurun_out/${TAG}_tmp.txt 2>&1
  python -c "
import json
for l in open('gpurun_out/${TAG}_tmp.txt'):
    if l.startswith('{\"config'):
        d=json.loads(l); print('$f'.split('/')[-1], {k: round(v,3) for k,v in d['ms'].items()}, round(d['fps'],1))
" | tee -a gpurun_out/${TAG}.txt
done
done
