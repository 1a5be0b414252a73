cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_ns_gpu.py -x -q > gpurun_out/pytest_ns.log 2>&1; tail -2 gpurun_out/pytest_ns.log
python tools/probe_ns.py --config ns2000 2>&1 | tail -3
python tools/probe_ns.py --config ns2000 --cold 1 2>&1 | tail -2
python tools/probe_ns.py --config cfg2 2>&1 | tail -2
BENCHES="ns2000" EXTRA="" bash tools/gpu_r2_bench.sh 2>&1 | grep -i "value\|fused\|all inter"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ns_sweep -s 3 -c 1 -o gpurun_out/prof_ns_sweep2 python tools/prof_eval.py --config ns2000 --mask ns --reps 6 > gpurun_out/prof_ns_sweep.log 2>&1
