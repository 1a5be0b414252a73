cd $GRAFT_REPO_ROOT
bash tools/gpu_r2_tests.sh
BENCHES="cfg2 ns2000 cfg3r2" bash tools/gpu_r2_bench.sh
