# K3 small-slab A/B: librsr.so vs experiment builds (librsr_*.so), one line per case and lib
cd ${GRAFT_REPO_ROOT:-/root/repo}
for c in ${CASES:-"8 609 1240 30 4 0.0" "8 720 1280 62 6 0.0" "8 720 1280 64 6 0.0" "8 720 1280 8 6 0.0"}; do
  REPS=10 python tools/k3_bench.py $c
  for f in paper_1807_07433_b200/librsr_*.so; do [ -e "$f" ] && RSR_LIB=$f REPS=10 python tools/k3_bench.py $c; done
done
