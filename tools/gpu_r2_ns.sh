cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1 || { tail -20 gpurun_out/smoke.log; exit 1; }
timeout 1500 python -m pytest tests/test_ns_gpu.py -x -q --durations=10 > gpurun_out/pytest_ns.log 2>&1; tail -15 gpurun_out/pytest_ns.log
BENCHES="ns2000 cfg2" bash tools/gpu_r2_bench.sh
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ns_sweep -s 3 -c 1 -o gpurun_out/prof_ns_sweep python tools/prof_eval.py --config ns2000 --mask ns --reps 6 > gpurun_out/prof_ns_sweep.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_ns_sweep.csv python tools/prof_eval.py --config ns2000 --mask ns --reps 6 > /dev/null 2>&1
grep k_ns gpurun_out/launches_ns_sweep.csv | tail -3
