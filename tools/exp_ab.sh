# K3 A/B of experiment builds (tools/): librsr.so without and with the partial maxima, then librsr_x*.so
cd ${GRAFT_REPO_ROOT:-/root/repo}
C=${C:-"8 720 1280 64 6 0.0"}
for i in 1 2; do
REPS=10 python tools/k3_bench.py $C
K3_WTA=1 REPS=10 python tools/k3_bench.py $C
for f in paper_1807_07433_b200/librsr_x*.so; do RSR_LIB=$f K3_WTA=1 REPS=10 python tools/k3_bench.py $C; done
done
