# A/B of experiment builds through bench.py: librsr.so and every librsr_*.so, twice
cd ${GRAFT_REPO_ROOT:-/root/repo}
for i in 1 2; do
for f in paper_1807_07433_b200/librsr.so paper_1807_07433_b200/librsr_*.so; do
  [ -e "$f" ] || continue
  RSR_LIB=$f python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$f', round(d['value'],1), d['kernel_ms'])"
done
done
