#!/bin/bash
# Parity tests + bench (+ optional ncu) on one GPU.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-q}
timeout ${PYT_TIMEOUT:-900} python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} ${PYK:+-k "$PYK"} > gpurun_out/${TAG}_pytest_gpu.log 2>&1; rc=$?
echo "pytest rc=$rc" >> gpurun_out/${TAG}_pytest_gpu.log; tail -30 gpurun_out/${TAG}_pytest_gpu.log
[ $rc -ne 0 ] && [ -z "$BENCH_ANYWAY" ] && exit 1
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
cat gpurun_out/${TAG}_bench.json; tail -5 gpurun_out/${TAG}_bench.err
if [ -n "$NCU" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/${TAG}_ncu_launches.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${NCU_KERNEL:-k_aggregate} -s ${NCU_SKIP:-2} -c 1 \
  -o gpurun_out/${TAG}_prof -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu2 rc=$?"
fi
