#!/bin/bash
# --set full pages of the dominant kernel of the remaining bench lines (issue-active / instructions evidence)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_inter_fast -s 2 -c 1 -o gpurun_out/fin_inter_cfg4 -f python tools/prof_dev.py --config cfg4 --steps 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_inter_fast -s 4 -c 1 -o gpurun_out/fin_inter_cfg3 -f python tools/prof_dev.py --config cfg3 --steps 6 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_inter_fast -s 4 -c 1 -o gpurun_out/fin_inter_cfg3r2 -f python tools/prof_dev.py --config cfg3r2 --steps 6 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_inter_fast -s 4 -c 1 -o gpurun_out/fin_inter_ns2000 -f python tools/prof_dev.py --config ns2000 --steps 6 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_inter -s 4 -c 1 -o gpurun_out/fin_inter_cfg3f -f python tools/prof_dev.py --config cfg3f --steps 6 > /dev/null 2>&1
for r in fin_inter_cfg4 fin_inter_cfg3 fin_inter_cfg3r2 fin_inter_ns2000 fin_inter_cfg3f; do python tools/ncu_summary.py gpurun_out/$r.ncu-rep gpurun_out/r02_ncu_${r#fin_}_final.csv; done
rm -f gpurun_out/fin_*.ncu-rep
