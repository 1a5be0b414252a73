#!/bin/bash
# ncu --set full of k_etga during device-resident ETGA steps (cfg4 and ns2000, theta=20)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in cfg4 ns2000; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_etga -s 3 -c 1 \
    -o gpurun_out/prof_etga_$c python tools/prof_dev.py --config $c --granular 20 --steps 6 > gpurun_out/prof_etga_$c.log 2>&1
done
ls -la gpurun_out/prof_etga_*.ncu-rep
