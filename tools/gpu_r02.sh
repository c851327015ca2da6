#!/bin/bash
# Round-2 GPU pass: full parity suite (no -x), bench N=1 plain and through the torchrun
# spawn path (NCCL process group + gather on one GPU).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r02}
timeout ${PYT_TIMEOUT:-1200} python -m pytest tests -m gpu -q ${PYK:+-k "$PYK"} > gpurun_out/${TAG}_pytest_gpu.log 2>&1; rc=$?
echo "pytest rc=$rc" >> gpurun_out/${TAG}_pytest_gpu.log; tail -15 gpurun_out/${TAG}_pytest_gpu.log
if [ -z "$NO_BENCH" ]; then
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
cat gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --spawn --steps 10 --no-cpu-baseline > gpurun_out/${TAG}_bench_spawn.json 2> gpurun_out/${TAG}_bench_spawn.err; echo "bench spawn rc=$?"
cat gpurun_out/${TAG}_bench_spawn.json; tail -3 gpurun_out/${TAG}_bench_spawn.err
fi
