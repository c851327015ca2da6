#!/bin/bash
# K2 iteration: cost-volume parity tests, per-phase times (c5, cP), default bench.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-k2}
timeout 900 python -m pytest tests -m gpu -x -q ${PYK:+-k "$PYK"} > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -3 gpurun_out/${TAG}_pytest.log
for c in "c5 8" "cP 8" "c1 8"; do timeout 300 python tools/phase_bench.py $c >> gpurun_out/${TAG}_phase.jsonl 2>>gpurun_out/${TAG}_phase.err; done
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
python - <<'P'
import json,os
t=os.environ.get("TAG","k2")
for l in open(f"gpurun_out/{t}_phase.jsonl"):
    d=json.loads(l); print(d["config"], {k: round(v,3) for k,v in d["ms"].items()}, round(d["fps"],1))
b=json.load(open(f"gpurun_out/{t}_bench.json")); print("bench", b["value"], b.get("e2e",{}).get("value"), b.get("clocks"))
P
