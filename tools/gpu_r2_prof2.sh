#!/bin/bash
# round-2 ncu evidence after the pick changes: launch list of bench.py cfg2 itself, --set full of the
# pick kernel (cfg2), of the penalised cfg2 inter kernel, and a cfg5 launch list
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_inter|k_pick" -c 240 --csv \
  --log-file gpurun_out/launches_bench_cfg2.csv python bench.py --steps 40 --warmup 3 --no-cpu-baseline --no-per-op --no-north-star --no-row-shard > gpurun_out/launches_bench_cfg2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pick_update1 -s 4 -c 1 -o gpurun_out/r02_pick_cfg2 -f python tools/prof_dev.py --config cfg2 --steps 6 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_inter_fast -s 4 -c 1 -o gpurun_out/r02_inter_pen_cfg2 -f python tools/prof_dev.py --config cfg2 --steps 6 --score penalised > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file gpurun_out/launches_bench_cfg5.csv python bench.py --config cfg5 --steps 4 --warmup 3 --no-cpu-baseline --no-per-op > gpurun_out/launches_bench_cfg5.log 2>&1
python tools/ncu_summary.py gpurun_out/r02_pick_cfg2.ncu-rep gpurun_out/r02_ncu_pick1_cfg2.csv
python tools/ncu_summary.py gpurun_out/r02_inter_pen_cfg2.ncu-rep gpurun_out/r02_ncu_inter_pen_cfg2.csv
ls -la gpurun_out/ | tail -12
