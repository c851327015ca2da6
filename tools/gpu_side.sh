#!/bin/bash
# Side benches (each prints JSON lines and a clock record): the paper's runtime sweep,
# the restricted band, the accuracy-evaluation kernels, the road model, the fused
# kernel vs the five calls, the restricted range on a sequence, the accuracy protocol.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-side}
for t in paper_sweep range_bench plane_bench road_bench match_bench range_seq accuracy_eval; do
  timeout 900 python tools/$t.py > gpurun_out/${TAG}_$t.jsonl 2> gpurun_out/${TAG}_$t.err; echo "$t rc=$?"
done
