cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/graph_floor tools/graph_floor.cu && /tmp/graph_floor > gpurun_out/graph_floor.txt 2>&1
nproc > gpurun_out/nproc.txt; grep "model name" /proc/cpuinfo | head -1 >> gpurun_out/nproc.txt
PROBE_MASK=ns python tools/probe_inter.py --config ns2000 > gpurun_out/probe_ns2000_ns.txt 2>&1
PROBE_MASK=ns python tools/probe_inter.py --config ns2000 --cold 0 > gpurun_out/probe_ns2000_ns_warm.txt 2>&1
PROBE_MASK=all python tools/probe_inter.py --config cfg2 > gpurun_out/probe_cfg2_all.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_ns_eval.csv python tools/prof_eval.py --config ns2000 --mask ns --reps 6 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_inter_fast -s 3 -c 1 -o gpurun_out/prof_ns_eval python tools/prof_eval.py --config ns2000 --mask ns --reps 6 > gpurun_out/prof_ns_eval.log 2>&1
cat gpurun_out/graph_floor.txt gpurun_out/probe_ns2000_ns*.txt
