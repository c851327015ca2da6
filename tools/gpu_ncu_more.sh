#!/bin/bash
# ncu --set full captures of the kernels the round evidence does not cover: K4
# (k_disparity) at c5, and the cP operating point's K2 (k_zncc_pair) and K3
# (k_aggregate_slide, the two-CTA small-slab instance) -- each only after the same
# bench command exited 0 without ncu.  One launch each (-s skips the warm-up launches).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-nm}
for c in c5 cP; do
  CMD="python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
  $CMD > gpurun_out/${TAG}_${c}_plain.log 2>&1; echo "$c plain rc=$?"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${TAG}_${c}_launches.csv $CMD > gpurun_out/${TAG}_${c}_ncu_launches.log 2>&1; echo "$c launches rc=$?"
done
C5="python bench.py --config c5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
CP="python bench.py --config cP --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_disparity -s 2 -c 1 \
  -o gpurun_out/${TAG}_k4_c5 -f $C5 > gpurun_out/${TAG}_k4_c5.log 2>&1; echo "k4 c5 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_zncc -s 2 -c 1 \
  -o gpurun_out/${TAG}_k2_cP -f $CP > gpurun_out/${TAG}_k2_cP.log 2>&1; echo "k2 cP rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_aggregate -s 4 -c 1 \
  -o gpurun_out/${TAG}_k3_cP -f $CP > gpurun_out/${TAG}_k3_cP.log 2>&1; echo "k3 cP rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_disparity -s 2 -c 1 \
  -o gpurun_out/${TAG}_k4_cP -f $CP > gpurun_out/${TAG}_k4_cP.log 2>&1; echo "k4 cP rc=$?"
