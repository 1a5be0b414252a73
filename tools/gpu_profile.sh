#!/bin/bash
# ncu evidence for profiles/: launch list of device-resident steps (cfg2, ns2000) and one
# --set full capture of the fused inter kernel and of the pick/update kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in cfg2 ns2000 cfg3r2; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$c.csv python tools/prof_dev.py --config $c --steps 6 > gpurun_out/launches_$c.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_inter_fast -s 4 -c 1 -o gpurun_out/prof_inter_cfg2 python tools/prof_dev.py --config cfg2 --steps 6 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_inter_fast -s 4 -c 1 -o gpurun_out/prof_inter_ns2000 python tools/prof_dev.py --config ns2000 --steps 6 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pick_update -s 4 -c 1 -o gpurun_out/prof_pick_cfg2 python tools/prof_dev.py --config cfg2 --steps 6 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_inter_fast -s 2 -c 1 -o gpurun_out/prof_inter_cfg4 python tools/prof_dev.py --config cfg4 --steps 3 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
