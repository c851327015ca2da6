#!/bin/bash
# Round evidence: the full -m gpu suite, the default bench (N=1) and through the
# torchrun spawn path (NCCL group + gather), the reference arm, the ncu launch list
# and one ncu --set full capture of the dominant kernel (K3) -- each ncu command only
# after the same command line exited 0 without ncu.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-ev}
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --spawn --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench_spawn.json 2> gpurun_out/${TAG}_bench_spawn.err; echo "spawn rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err; echo "ref rc=$?"
for c in c1 c2 c4 cP; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/${TAG}_bench_configs.jsonl 2>> gpurun_out/${TAG}_bench_configs.err; done; echo "configs rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1; echo "ncu1 rc=$?"
CMD1="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD1 > gpurun_out/${TAG}_plain1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${NCU_KERNEL:-k_aggregate} -s ${NCU_SKIP:-2} -c 1 \
  -o gpurun_out/${TAG}_k3 -f $CMD1 > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu2 rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/${TAG}_smoke.log
