#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pick_update1 -s 40 -c 1 -o gpurun_out/pick_cfg2 -f \
  python tools/probe_step.py --config ${CFG:-cfg2} --steps 6 --replicas 20 > gpurun_out/ncu_pick.log 2>&1
tail -3 gpurun_out/ncu_pick.log
