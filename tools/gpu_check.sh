#!/bin/bash
# One GPU pass: parity tests, bench, ncu launch list, ncu full capture of K3.
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r01}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
if [ -z "$NO_NCU" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/${TAG}_ncu_launches.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${NCU_KERNEL:-k_aggregate} -s ${NCU_SKIP:-2} -c 1 \
  -o gpurun_out/${TAG}_agg -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu2 rc=$?"
fi
