cd $GRAFT_REPO_ROOT
for R in ${RS:-0 144 180 240}; do
  if [ $R -eq 0 ]; then unset RSR_K3_ROWS; else export RSR_K3_ROWS=$R; fi
  python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('R=$R', round(d['value'],1), round(d['kernel_ms']['aggregate_pair'],3))"
done
